cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r31_topo.txt 2>&1
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r31_bench$N.log 2>&1
echo "rc=$?" >> gpurun_out/r31_bench$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 10 --warmup 3 --output sharded --e2e-steps 0 > gpurun_out/r31_bench${N}s.log 2>&1
echo "rc=$?" >> gpurun_out/r31_bench${N}s.log
done
timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r31_bench1.log 2>&1
