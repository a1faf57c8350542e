cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/w64b_pytest.log 2>&1; tail -2 gpurun_out/w64b_pytest.log
for wl in C3 sweep:35 sweep:39 sweep:47 sweep:51 sweep:55 sweep:59 sweep:63; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done
