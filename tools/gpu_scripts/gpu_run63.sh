cd $GRAFT_REPO_ROOT
timeout 300 python tools/phase_time.py C3 >> gpurun_out/r63.log 2>&1
GAR_COORD_LOADER=tma timeout 300 python tools/phase_time.py C3 >> gpurun_out/r63.log 2>&1
timeout 300 python tools/phase_time.py sweep:15 >> gpurun_out/r63.log 2>&1
