cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -k "average or multi_krum or bulyan or smoke" > gpurun_out/at_pytest.log 2>&1; tail -2 gpurun_out/at_pytest.log
for n in 7 11 15 35 47 63; do timeout 300 python tools/ab_step.py sweep:$n 2>&1 | tail -1; done
