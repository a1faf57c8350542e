cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/prof_step.py > gpurun_out/p27_plain.log 2>&1 && \
timeout 1500 $NCU --set full --clock-control none --import-source on -k "regex:gram_tc|coord_select|coord_ldg|copy_row" -s 9 -c 9 -o gpurun_out/p27_full python tools/prof_step.py > gpurun_out/p27_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/p27_plain.log
