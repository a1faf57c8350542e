cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pf2_pytest.log 2>&1; tail -2 gpurun_out/pf2_pytest.log
for rep in 1 2; do
timeout 900 python bench.py > gpurun_out/pf2_bench_$rep.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/pf2_bench_$rep.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', j['ms_per_step'], j['value'], j['roofline']['frac'], {r:v['ms'] for r,v in j['per_rule'].items()}, j['clocks'])"
done
