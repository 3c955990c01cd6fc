# trace + parity of library variants built with experiment knobs: usage TAG CONFIG variant...
cd $GRAFT_REPO_ROOT
TAG=$1; C=$2; shift 2
L=paper_1411_4356_b200
cp $L/libss_b200.so /tmp/libss_keep.so
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_base_$C.json 2> gpurun_out/${TAG}_base_$C.err
for v in "$@"; do
  cp $L/libss_b200_$v.so $L/libss_b200.so
  timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_${v}_$C.json 2> gpurun_out/${TAG}_${v}_$C.err
  timeout 600 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity" > gpurun_out/${TAG}_${v}_tests.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_${v}_bench.json 2> gpurun_out/${TAG}_${v}_bench.err
done
cp /tmp/libss_keep.so $L/libss_b200.so
echo done
