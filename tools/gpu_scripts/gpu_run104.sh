cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 tools/check_ingress.py C3 > gpurun_out/r104_2.log 2>&1; echo "rc=$?" >> gpurun_out/r104_2.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r104_pytest.log 2>&1; tail -2 gpurun_out/r104_pytest.log >> gpurun_out/r104_2.log
