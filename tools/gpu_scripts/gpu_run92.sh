cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r92_check.log 2>&1; echo "rc=$?" >> gpurun_out/r92_check.log; cat gpurun_out/r92_check.log
for v in base ""; do GAR_LIB_VARIANT=$v timeout 300 python tools/gram_time.py 3 5 7 8 >> gpurun_out/r92.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r92_pytest.log 2>&1; tail -3 gpurun_out/r92_pytest.log
timeout 300 python tools/ab_step.py sweep:7 >> gpurun_out/r92.log 2>&1
