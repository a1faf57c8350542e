cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r21_bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r21_bench1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r21_bench2.log 2>&1
echo "bench2 rc=$?" >> gpurun_out/r21_bench2.log
