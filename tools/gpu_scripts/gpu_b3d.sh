cd $GRAFT_REPO_ROOT
for wl in C3 C4; do for rep in 1 2 3; do
GAR_BULYAN_B3_OFF=1 timeout 300 python tools/bulyan_ctx.py $wl 2>&1 | tail -1
timeout 300 python tools/bulyan_ctx.py $wl 2>&1 | tail -1
done; done
for rep in 1 2; do
GAR_BULYAN_B3_OFF=1 timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3d_off_$rep.log 2>&1; tail -1 gpurun_out/b3d_off_$rep.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 off', j['ms_per_step'], j['per_rule']['bulyan']['ms'])"
timeout 900 python bench.py --e2e-steps 0 --no-cpu-baseline > gpurun_out/b3d_prod_$rep.log 2>&1; tail -1 gpurun_out/b3d_prod_$rep.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3 prod', j['ms_per_step'], j['per_rule']['bulyan']['ms'])"
done
