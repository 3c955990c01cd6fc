# bench (default workload) + ncu launch list + one ncu --set full capture of k_chain_trsv.
# usage (under gpurun): bash scripts/gpu_profile.sh TAG [bench args...]
cd $GRAFT_REPO_ROOT
TAG=$1; shift
python bench.py --steps 5 --warmup 3 "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python bench.py --steps 2 --warmup 1 --dims "" --no-cpu-baseline "$@" > gpurun_out/${TAG}_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 --dims "" --no-cpu-baseline "$@" > gpurun_out/${TAG}_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_chain_trsv -s 6 -c 2 -o gpurun_out/${TAG}_trsv \
    python bench.py --steps 2 --warmup 1 --dims "" --no-cpu-baseline "$@" > gpurun_out/${TAG}_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 3 -c 1 -o gpurun_out/${TAG}_spmv \
    python bench.py --steps 2 --warmup 1 --dims "" --no-cpu-baseline "$@" > gpurun_out/${TAG}_ncu3.log 2>&1
echo done
