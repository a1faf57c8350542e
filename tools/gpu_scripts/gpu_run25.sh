cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r25_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r25_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r25_bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r25_bench1.log
for wl in C3 sweep:63 C2 C1; do timeout 300 python tools/ab_step.py $wl >> gpurun_out/r25_ab.log 2>&1; done
