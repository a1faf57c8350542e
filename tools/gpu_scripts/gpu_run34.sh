cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r34_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r34_check_gram.log
for wl in C3 sweep:7 sweep:11 sweep:15 sweep:19 C1 C2; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r34_ab.log 2>&1; done
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r34_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r34_pytest_gpu.log
