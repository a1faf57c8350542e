cd $GRAFT_REPO_ROOT
for wl in C1 C2; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r72.log 2>&1; timeout 300 python tools/phase_time.py $wl >> gpurun_out/r72.log 2>&1; done
