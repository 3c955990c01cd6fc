# iteration call: substitution/steady-state parity tests, default bench, trace; extra commands in $EXTRA
cd $GRAFT_REPO_ROOT
TAG=$1
timeout 900 python -m pytest tests -m gpu -x -q -k "subst or steady_state or multi_cycle or full_size_medium or sm_budget or concurrent" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_trace_medium.json 2> gpurun_out/${TAG}_trace_medium.err
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/${TAG}_extra.log 2>&1; fi
echo done
