cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/check_fused.py > gpurun_out/r32_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r32_fused.log
for o in fused replicated sharded; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 10 --warmup 3 --output $o --e2e-steps 0 > gpurun_out/r32_bench2_$o.log 2>&1
echo "rc=$?" >> gpurun_out/r32_bench2_$o.log
done
