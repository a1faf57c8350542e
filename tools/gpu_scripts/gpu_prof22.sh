cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/prof_step.py > gpurun_out/p22_plain.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p22_launches.csv python tools/prof_step.py > gpurun_out/p22_ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/p22_plain.log
timeout 1500 $NCU --set full --clock-control none --import-source on -k "regex:gram_tc|coord_select|copy_row" -s 9 -c 9 -o gpurun_out/p22_full python tools/prof_step.py > gpurun_out/p22_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/p22_plain.log
