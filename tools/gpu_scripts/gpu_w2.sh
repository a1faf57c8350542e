cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -k "trimmed or loader or every_n or fullsize or smoke" > gpurun_out/w2_pytest.log 2>&1; tail -2 gpurun_out/w2_pytest.log
for wl in C3 sweep:19 sweep:23 sweep:27 C4; do for rep in 1 2; do
timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
GAR_COORD_LOADER=tma timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1
done; done
