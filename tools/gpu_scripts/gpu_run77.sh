cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_fullsize_gpu.py -m gpu -v -rA > gpurun_out/r77_full.log 2>&1; tail -15 gpurun_out/r77_full.log
