# round-2 call: the stale-shared-memory regression test on the pre-fix build (expected to FAIL) and on the
# default build (expected to pass); chain variants (trace + parity + bench on configs[2]); the 64-point sweep
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
L=paper_1411_4356_b200
cp $L/libss_b200.so /tmp/libss_keep.so
cp $L/libss_b200_prefix.so $L/libss_b200.so
timeout 600 python -m pytest tests -m gpu -q -k "stale_shared" > gpurun_out/${TAG}_prefix_stale.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_prefix_stale.log
cp /tmp/libss_keep.so $L/libss_b200.so
timeout 600 python -m pytest tests -m gpu -q -k "stale_shared or concurrent_points or sm_budget" > gpurun_out/${TAG}_default_stale.log 2>&1; echo "rc $?" >> gpurun_out/${TAG}_default_stale.log
for v in "$@"; do
  cp $L/libss_b200_$v.so $L/libss_b200.so
  timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_${v}_trace.json 2> gpurun_out/${TAG}_${v}_trace.err
  timeout 900 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity or medium or stale_shared" > gpurun_out/${TAG}_${v}_tests.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_${v}_bench.json 2> gpurun_out/${TAG}_${v}_bench.err
done
cp /tmp/libss_keep.so $L/libss_b200.so
timeout 1500 python bench.py --workload sweep --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_sweep.json 2> gpurun_out/${TAG}_bench_sweep.err
echo done
