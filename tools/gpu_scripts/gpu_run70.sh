cd $GRAFT_REPO_ROOT
for o in fused fused-p2p sharded; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --output $o --no-cpu-baseline > gpurun_out/r70_bench_$o.log 2>&1; done
