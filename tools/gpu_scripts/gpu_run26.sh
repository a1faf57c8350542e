cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r26_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r26_check_gram.log
for wl in C3 sweep:63 sweep:7 C2 C1; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r26_ab.log 2>&1; done
GAR_COORD_LOADER=tma timeout 300 python tools/ab_step.py C3 >> gpurun_out/r26_ab.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r26_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r26_pytest_gpu.log
