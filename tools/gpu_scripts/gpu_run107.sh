cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r107.log 2>&1; tail -2 gpurun_out/r107.log
