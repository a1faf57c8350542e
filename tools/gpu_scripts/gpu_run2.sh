cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r3_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r3_check_gram.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r3_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r3_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r3_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r3_bench.log
