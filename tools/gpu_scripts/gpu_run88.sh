cd $GRAFT_REPO_ROOT
timeout 600 python tools/mda_time.py > gpurun_out/r88.log 2>&1
