cd $GRAFT_REPO_ROOT
TAG=$1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/memcheck_small.py conc > gpurun_out/${TAG}_memcheck.log 2>&1
timeout 1200 python scripts/sweep_race.py 30 64 4 lock_setup 2 > gpurun_out/${TAG}_race_lock_setup.jsonl 2> gpurun_out/${TAG}_race_lock_setup.err
bash scripts/gpu_variants.sh $TAG medium dl dl1280
echo done
