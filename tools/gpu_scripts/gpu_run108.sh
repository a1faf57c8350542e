cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r108.log 2>&1; tail -20 gpurun_out/r108.log
