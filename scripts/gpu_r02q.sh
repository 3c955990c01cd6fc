# round-2 call: more variants (trace + parity + bench on configs[2])
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
L=paper_1411_4356_b200
cp $L/libss_b200.so /tmp/libss_keep.so
for v in "$@"; do
  cp $L/libss_b200_$v.so $L/libss_b200.so
  timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_${v}_trace.json 2> gpurun_out/${TAG}_${v}_trace.err
  timeout 900 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity or medium or stale_shared" > gpurun_out/${TAG}_${v}_tests.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_${v}_bench.json 2> gpurun_out/${TAG}_${v}_bench.err
done
cp /tmp/libss_keep.so $L/libss_b200.so
echo done
