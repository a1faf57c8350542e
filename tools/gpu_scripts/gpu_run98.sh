cd $GRAFT_REPO_ROOT
timeout 900 python tools/paper_protocol.py > gpurun_out/r98.log 2>&1
