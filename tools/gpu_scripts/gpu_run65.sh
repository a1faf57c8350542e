cd $GRAFT_REPO_ROOT
timeout 300 python tools/phase_time.py C3 >> gpurun_out/r65.log 2>&1
