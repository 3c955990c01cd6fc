# round-2 GPU call: full GPU suite, profile of the default bench, then configs[3] probes
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/g3_host.txt
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/g3_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/g3_tests.log
bash scripts/gpu_profile.sh g3
SSB_ILUT_PROF=1 timeout 1800 python scripts/sweep_probe.py large - "1e-4:80:0.01" 1e-15 > gpurun_out/g3_large.jsonl 2> gpurun_out/g3_large.err
