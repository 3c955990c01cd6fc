# round-2 GPU call: full GPU suite, profile of the default bench (configs[2]), the configs[4] sweep bench
cd $GRAFT_REPO_ROOT
TAG=${1:-r02a}
nproc > gpurun_out/${TAG}_host.txt; free -g >> gpurun_out/${TAG}_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${TAG}_tests.log
timeout 1500 bash scripts/gpu_profile.sh ${TAG}
timeout 1500 python bench.py --workload sweep --steps 1 --warmup 1 > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err
echo done
