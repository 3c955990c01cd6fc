# round-2 final evidence call on the default build: full GPU suite, smoke, default bench, ncu launch list,
# one ncu --set full capture of k_chain_trsv (raw page exported as CSV for profiles/)
cd $GRAFT_REPO_ROOT
TAG=$1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python scripts/trace_trsv.py medium > gpurun_out/${TAG}_trace_medium.json 2> gpurun_out/${TAG}_trace_medium.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_trsv -s 6 -c 2 -o gpurun_out/${TAG}_trsv \
  python bench.py --steps 2 --warmup 1 --dims "" --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
ncu -i gpurun_out/${TAG}_trsv.ncu-rep --page raw --csv > gpurun_out/${TAG}_trsv_raw.csv 2>/dev/null
rm -f gpurun_out/${TAG}_trsv.ncu-rep
echo done
