cd $GRAFT_REPO_ROOT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/check_fused.py > gpurun_out/r79_check.log 2>&1; echo "check rc=$?" >> gpurun_out/r79_check.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r79_bench.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r79_bench2.log 2>&1
