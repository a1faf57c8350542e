cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -k "bulyan or mean_around" > gpurun_out/b3a_pytest.log 2>&1; tail -2 gpurun_out/b3a_pytest.log
for wl in C3 C4; do
for rep in 1 2; do
GAR_BULYAN_B3_OFF=1 timeout 300 python tools/phase_time.py $wl > gpurun_out/b3a_off_${wl}_$rep.log 2>&1; echo "off $wl $(grep -o '"combine_bulyan": [0-9.]*' gpurun_out/b3a_off_${wl}_$rep.log)"
timeout 300 python tools/phase_time.py $wl > gpurun_out/b3a_prod_${wl}_$rep.log 2>&1; echo "prod $wl $(grep -o '"combine_bulyan": [0-9.]*' gpurun_out/b3a_prod_${wl}_$rep.log)"
for v in minb5 lds ldsminb5 ldsminb6; do
GAR_LIB_VARIANT=$v timeout 300 python tools/phase_time.py $wl > gpurun_out/b3a_${v}_${wl}_$rep.log 2>&1; echo "$v $wl $(grep -o '"combine_bulyan": [0-9.]*' gpurun_out/b3a_${v}_${wl}_$rep.log)"
done; done; done
