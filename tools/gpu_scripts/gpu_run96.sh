cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r96_b1.log 2>&1; grep '^{' gpurun_out/r96_b1.log | tail -1 | head -c 300; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r96_b2.log 2>&1; grep '^{' gpurun_out/r96_b2.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['gpu_launches'], d['steps'])"
