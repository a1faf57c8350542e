cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r60_pytest.log 2>&1; tail -3 gpurun_out/r60_pytest.log
for wl in sweep:7 sweep:11 sweep:15 sweep:19 sweep:23 sweep:27 C3; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r60_ab.log 2>&1; done
