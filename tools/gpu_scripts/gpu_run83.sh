cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_step.py C1 > gpurun_out/r83_plain.log 2>&1 && \
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/r83_launches.csv python tools/ab_step.py C1 > gpurun_out/r83_ncu.log 2>&1
echo rc=$? >> gpurun_out/r83_plain.log
