cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 300 python tools/prof_step.py > gpurun_out/p1_plain.log 2>&1 && \
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p1_launches.csv python tools/prof_step.py > gpurun_out/p1_ncu_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/p1_plain.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gram_tc -s 3 -c 1 -o gpurun_out/p1_gram python tools/prof_step.py > gpurun_out/p1_ncu_gram.log 2>&1
echo "gram rc=$?" >> gpurun_out/p1_plain.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:coord_select -s 7 -c 2 -o gpurun_out/p1_coord python tools/prof_step.py > gpurun_out/p1_ncu_coord.log 2>&1
echo "coord rc=$?" >> gpurun_out/p1_plain.log
