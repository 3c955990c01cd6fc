cd $GRAFT_REPO_ROOT
TAG=$1
L=paper_1411_4356_b200
timeout 900 python scripts/sweep_race.py 30 64 4 full 3 > gpurun_out/${TAG}_race_full.jsonl 2> gpurun_out/${TAG}_race_full.err
timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_trace_medium.json 2> gpurun_out/${TAG}_trace_medium.err
timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
cp $L/libss_b200.so /tmp/libss_keep.so
cp $L/libss_b200_ldg.so $L/libss_b200.so
timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_ldg_medium.json 2> gpurun_out/${TAG}_ldg_medium.err
timeout 600 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity" > gpurun_out/${TAG}_ldg_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_ldg_bench.json 2> gpurun_out/${TAG}_ldg_bench.err
cp /tmp/libss_keep.so $L/libss_b200.so
echo done
