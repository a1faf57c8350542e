cd $GRAFT_REPO_ROOT
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/check_fused.py > gpurun_out/r69_check.log 2>&1; echo "check rc=$?" >> gpurun_out/r69_check.log
for o in fused fused-p2p sharded; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --steps 10 --warmup 3 --output $o --no-cpu-baseline > gpurun_out/r69_bench_$o.log 2>&1; done
