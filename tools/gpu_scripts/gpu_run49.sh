cd $GRAFT_REPO_ROOT
timeout 120 tools/tmembench > gpurun_out/r49.log 2>&1
