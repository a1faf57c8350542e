cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r56_pytest.log 2>&1; tail -3 gpurun_out/r56_pytest.log
for wl in C3 sweep:15 sweep:47 sweep:63; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r56_ab.log 2>&1; done
