# round-2 re-entry validation call: full GPU suite, smoke, default bench, per-step trace of configs[2]
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_trace_medium.json 2> gpurun_out/${TAG}_trace_medium.err
echo done
