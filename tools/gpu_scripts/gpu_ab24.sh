cd $GRAFT_REPO_ROOT
for wl in C3 sweep:63 sweep:7 C2; do
timeout 300 python tools/ab_step.py $wl >> gpurun_out/ab24.log 2>&1
GAR_COORD_LOADER=ldg timeout 300 python tools/ab_step.py $wl >> gpurun_out/ab24.log 2>&1
done
GAR_COORD_LOADER=ldg timeout 900 python -m pytest tests/test_parity_gpu.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/ab24_pytest_ldg.log 2>&1
echo "rc=$?" >> gpurun_out/ab24_pytest_ldg.log
