cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r87_pytest.log 2>&1; tail -8 gpurun_out/r87_pytest.log
