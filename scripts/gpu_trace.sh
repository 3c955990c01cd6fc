# per-block critical-path stamps of the block substitution (scripts/trace_trsv.py) on given configs
cd $GRAFT_REPO_ROOT
TAG=$1; shift
for c in "$@"; do timeout 900 python scripts/trace_trsv.py $c > gpurun_out/${TAG}_trace_$c.json 2> gpurun_out/${TAG}_trace_$c.err; done
echo done
