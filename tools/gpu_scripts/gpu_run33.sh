cd $GRAFT_REPO_ROOT
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r33_bench$N.log 2>&1
echo "rc=$?" >> gpurun_out/r33_bench$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 5 --warmup 3 --workload C4 --e2e-steps 0 > gpurun_out/r33_c4_$N.log 2>&1
echo "rc=$?" >> gpurun_out/r33_c4_$N.log
done
timeout 900 python bench.py --steps 5 --warmup 3 --workload C4 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r33_c4_1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/check_fused.py > gpurun_out/r33_fused4.log 2>&1
echo "rc=$?" >> gpurun_out/r33_fused4.log
