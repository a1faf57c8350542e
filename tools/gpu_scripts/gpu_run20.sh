cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r20_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r20_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r20_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r20_bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r20_bench1.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r20_bench2.log 2>&1
echo "bench2 rc=$?" >> gpurun_out/r20_bench2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 --output sharded --e2e-steps 0 > gpurun_out/r20_bench2s.log 2>&1
echo "bench2s rc=$?" >> gpurun_out/r20_bench2s.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r20_ref.log 2>&1
echo "ref rc=$?" >> gpurun_out/r20_ref.log
