cd $GRAFT_REPO_ROOT
timeout 120 tools/mmabench > gpurun_out/r50.log 2>&1
