cd $GRAFT_REPO_ROOT
timeout 300 python tools/drift.py 25 > gpurun_out/r67.log 2>&1
