cd $GRAFT_REPO_ROOT
timeout 300 python tools/gram_prof.py 7 31 63 > gpurun_out/r41.log 2>&1
