cd $GRAFT_REPO_ROOT
for o in replicated-async fused fused-mc replicated; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --output $o --no-cpu-baseline --e2e-steps 0 > gpurun_out/r71_bench_$o.log 2>&1; done
