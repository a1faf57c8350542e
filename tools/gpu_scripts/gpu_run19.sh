cd $GRAFT_REPO_ROOT
timeout 300 python tools/check_gram.py > gpurun_out/r19_check_gram.log 2>&1; echo "rc=$?" >> gpurun_out/r19_check_gram.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r19_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r19_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r19_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r19_bench.log
timeout 300 python tools/prof_step.py > gpurun_out/r19_plain.log 2>&1 && \
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:coord_select -s 6 -c 6 -o gpurun_out/r19_coord python tools/prof_step.py > gpurun_out/r19_ncu_coord.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r19_plain.log
