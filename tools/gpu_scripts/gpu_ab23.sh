cd $GRAFT_REPO_ROOT
timeout 300 python tools/ab_step.py > gpurun_out/ab23.log 2>&1
GAR_L2_EVICT_FIRST=0 timeout 300 python tools/ab_step.py >> gpurun_out/ab23.log 2>&1
timeout 300 python tools/ab_step.py sweep:63 >> gpurun_out/ab23.log 2>&1
GAR_L2_EVICT_FIRST=0 timeout 300 python tools/ab_step.py sweep:63 >> gpurun_out/ab23.log 2>&1
timeout 300 python tools/ab_step.py sweep:7 >> gpurun_out/ab23.log 2>&1
