cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r90_pytest.log 2>&1; tail -3 gpurun_out/r90_pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 tools/check_fused.py > gpurun_out/r90_check.log 2>&1; echo "check rc=$?"
