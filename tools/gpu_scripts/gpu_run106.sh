cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -x -q -k "exchange_single or raw_address" > gpurun_out/r106.log 2>&1; tail -15 gpurun_out/r106.log
