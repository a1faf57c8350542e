cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r64_pytest.log 2>&1; tail -3 gpurun_out/r64_pytest.log
timeout 300 python tools/phase_time.py C3 >> gpurun_out/r64.log 2>&1
for wl in C3 sweep:7 sweep:15 sweep:35 sweep:63; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r64.log 2>&1; done
