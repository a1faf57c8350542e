cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/check_fused.py > gpurun_out/r113.log 2>&1; echo "check rc=$?" >> gpurun_out/r113.log; grep -E "mda|around|rc=" gpurun_out/r113.log | head
