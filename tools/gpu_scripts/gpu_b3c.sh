cd $GRAFT_REPO_ROOT
for wl in C3 C4; do for il in 0 1; do
INTERLEAVE=$il GAR_BULYAN_B3_OFF=1 timeout 300 python tools/bulyan_ctx.py $wl 2>&1 | tail -1
INTERLEAVE=$il timeout 300 python tools/bulyan_ctx.py $wl 2>&1 | tail -1
done; done
GAR_BULYAN_B3_OFF=1 timeout 900 python bench.py --workload C4 > gpurun_out/b3c_bench_C4_off.log 2>&1; tail -1 gpurun_out/b3c_bench_C4_off.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C4 off', j['ms_per_step'], {r:v['ms'] for r,v in j['per_rule'].items()})"
timeout 900 python bench.py --workload C4 > gpurun_out/b3c_bench_C4.log 2>&1; tail -1 gpurun_out/b3c_bench_C4.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C4 prod', j['ms_per_step'], {r:v['ms'] for r,v in j['per_rule'].items()})"
