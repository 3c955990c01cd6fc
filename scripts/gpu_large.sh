# configs[3] at full size under the reading of DESIGN.md R14 (n_th = 1e-15, larger fill), then the sweep bench
cd $GRAFT_REPO_ROOT
TAG=$1; COMBOS=${2:-"1e-5:150:0.01"}
timeout 1500 python bench.py --workload sweep --steps 1 --warmup 1 > gpurun_out/${TAG}_sweep.json 2> gpurun_out/${TAG}_sweep.err
SSB_SETUP_PROF=1 timeout 4000 python scripts/sweep_probe.py large - "$COMBOS" 1e-15 > gpurun_out/${TAG}_large.jsonl 2> gpurun_out/${TAG}_large.err
free -g >> gpurun_out/${TAG}_large.err
echo done
