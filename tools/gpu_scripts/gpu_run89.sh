cd $GRAFT_REPO_ROOT
timeout 1200 python tools/sweep.py > gpurun_out/r89_sweep.md 2>&1; echo "rc=$?" >> gpurun_out/r89_sweep.md
