cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/r57_bench.log 2>&1; tail -c 3000 gpurun_out/r57_bench.log
