# sweep with more points in flight per GPU (host-bound setups): free memory before, bench line
cd $GRAFT_REPO_ROOT
TAG=$1; C=$2
mkdir -p gpurun_out
free -g > gpurun_out/${TAG}_free.txt; nproc >> gpurun_out/${TAG}_free.txt
( while true; do free -g | sed -n 2p; sleep 20; done ) > gpurun_out/${TAG}_mem_watch.txt 2>&1 &
W=$!
timeout 1300 python bench.py --workload sweep --steps 1 --warmup 1 --concurrent $C > gpurun_out/${TAG}_bench_sweep_c$C.json 2> gpurun_out/${TAG}_bench_sweep_c$C.err
kill $W
echo done
