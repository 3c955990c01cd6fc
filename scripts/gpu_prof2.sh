# critical-path profiles of the block substitution on one config: globaltimer trace, then the
# lieutenant and chain-team cycle profiles (profiling builds swapped in, then restored)
cd $GRAFT_REPO_ROOT
TAG=$1; C=${2:-medium}
L=paper_1411_4356_b200
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_trace_$C.json 2> gpurun_out/${TAG}_trace_$C.err
cp $L/libss_b200.so /tmp/libss_keep.so
cp $L/libss_b200_ltprof.so $L/libss_b200.so
timeout 600 python scripts/trace_lt.py $C > gpurun_out/${TAG}_lt_$C.json 2> gpurun_out/${TAG}_lt_$C.err
cp $L/libss_b200_teamprof.so $L/libss_b200.so
timeout 600 python scripts/trace_team.py $C > gpurun_out/${TAG}_team_$C.json 2> gpurun_out/${TAG}_team_$C.err
cp $L/libss_b200_noq.so $L/libss_b200.so
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_noq_$C.json 2> gpurun_out/${TAG}_noq_$C.err
cp $L/libss_b200_kd3.so $L/libss_b200.so
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_kd3_$C.json 2> gpurun_out/${TAG}_kd3_$C.err
timeout 600 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity" > gpurun_out/${TAG}_kd3_tests.log 2>&1
cp $L/libss_b200_g3w.so $L/libss_b200.so
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_g3w_$C.json 2> gpurun_out/${TAG}_g3w_$C.err
timeout 600 python -m pytest tests -m gpu -x -q -k "subst or steady_state_parity" > gpurun_out/${TAG}_g3w_tests.log 2>&1
cp $L/libss_b200_push3.so $L/libss_b200.so
timeout 600 python scripts/trace_trsv.py $C > gpurun_out/${TAG}_push3_$C.json 2> gpurun_out/${TAG}_push3_$C.err
cp /tmp/libss_keep.so $L/libss_b200.so
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > gpurun_out/${TAG}_extra.log 2>&1; fi
echo done
