cd $GRAFT_REPO_ROOT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_mc.py > gpurun_out/r68.log 2>&1
nvidia-smi topo -m >> gpurun_out/r68.log 2>&1
