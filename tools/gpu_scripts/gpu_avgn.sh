cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -k "average or multi_krum or smoke or every_n or every_family" > gpurun_out/an_pytest.log 2>&1; tail -2 gpurun_out/an_pytest.log
for n in 7 11 15 35 63; do for rep in 1 2; do
GAR_AVG_RUNTIME_R=1 timeout 300 python tools/ab_step.py sweep:$n 2>&1 | tail -1 | grep -o '"env.*"median": [0-9.]*'
timeout 300 python tools/ab_step.py sweep:$n 2>&1 | tail -1 | grep -o '"env.*"median": [0-9.]*'
done; done
for wl in C1 C2; do timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; GAR_AVG_RUNTIME_R=1 timeout 300 python tools/ab_step.py $wl 2>&1 | tail -1; done
