cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545 tools/check_ingress.py C3 > gpurun_out/r99_4.log 2>&1; echo "rc=$?" >> gpurun_out/r99_4.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29546 tools/check_ingress.py C3 > gpurun_out/r99_2.log 2>&1; echo "rc=$?" >> gpurun_out/r99_2.log
