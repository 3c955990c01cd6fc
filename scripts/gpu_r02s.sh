# round-2 evidence call: full GPU suite, default bench, smoke, concurrent-sweep race diagnostic, launch list
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python scripts/sweep_race.py 30 32 4 full 2 > gpurun_out/${TAG}_race_full.jsonl 2> gpurun_out/${TAG}_race_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo done
