cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "empty_and_degenerate" > gpurun_out/r109.log 2>&1; tail -30 gpurun_out/r109.log
