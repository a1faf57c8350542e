cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r86_pytest.log 2>&1; tail -3 gpurun_out/r86_pytest.log
timeout 300 python tools/server_step_time.py C3 >> gpurun_out/r86.log 2>&1
