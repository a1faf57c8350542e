cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r81_smoke.log 2>&1; tail -2 gpurun_out/r81_smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r81_ref.log 2>&1; tail -1 gpurun_out/r81_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r81_ref2.log 2>&1; echo "ref2 rc=$?"; grep '^{' gpurun_out/r81_ref2.log | tail -1 | head -c 300; echo
timeout 900 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r81_c4.log 2>&1; grep '^{' gpurun_out/r81_c4.log | tail -1 | head -c 400; echo
timeout 600 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r81_c2.log 2>&1; grep '^{' gpurun_out/r81_c2.log | tail -1 | head -c 300; echo
