cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --workload C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r93_c4_4.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --workload C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r93_c4_2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --workload C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --output sharded > gpurun_out/r93_c4_4s.log 2>&1
