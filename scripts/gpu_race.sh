cd $GRAFT_REPO_ROOT
TAG=$1
for m in full lock_solve lock_setup; do timeout 900 python scripts/sweep_race.py 30 64 4 $m 3 > gpurun_out/${TAG}_race_$m.jsonl 2> gpurun_out/${TAG}_race_$m.err; done
echo done
