cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545 tools/check_ingress.py C3 > gpurun_out/r100_4.log 2>&1; echo "rc=$?" >> gpurun_out/r100_4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/check_fused.py > gpurun_out/r100_check.log 2>&1; echo "check rc=$?" >> gpurun_out/r100_4.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r100_pytest.log 2>&1; tail -2 gpurun_out/r100_pytest.log >> gpurun_out/r100_4.log
