cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/b3b_pytest.log 2>&1; tail -2 gpurun_out/b3b_pytest.log
for wl in C3 C4 C2; do for rep in 1 2; do
GAR_BULYAN_B3_OFF=1 timeout 300 python tools/phase_time.py $wl > gpurun_out/b3b_off_${wl}_$rep.log 2>&1; echo "off $wl $(grep -o '"combine_bulyan": [0-9.]*' gpurun_out/b3b_off_${wl}_$rep.log)"
timeout 300 python tools/phase_time.py $wl > gpurun_out/b3b_prod_${wl}_$rep.log 2>&1; echo "prod $wl $(grep -o '"combine_bulyan": [0-9.]*' gpurun_out/b3b_prod_${wl}_$rep.log)"
done; done
for rep in 1 2; do
GAR_BULYAN_B3_OFF=1 timeout 300 python tools/ab_step.py C3 > gpurun_out/b3b_ab_off_$rep.log 2>&1; tail -1 gpurun_out/b3b_ab_off_$rep.log
timeout 300 python tools/ab_step.py C3 > gpurun_out/b3b_ab_prod_$rep.log 2>&1; tail -1 gpurun_out/b3b_ab_prod_$rep.log
done
timeout 900 python bench.py > gpurun_out/b3b_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/b3b_bench.log
