cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r35_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r35_check_gram.log
timeout 900 python tools/sweep.py > gpurun_out/r35_sweep.md 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r35_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r35_pytest_gpu.log
