cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_step.py > gpurun_out/r30.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/r30_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r30_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r30_bench1.log 2>&1
echo "bench rc=$?" >> gpurun_out/r30_bench1.log
timeout 1500 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k "regex:gram_tc|coord_select|coord_ldg|copy_row" -s 9 -c 9 -o gpurun_out/p30_full python tools/prof_step.py > gpurun_out/p30_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r30.log
