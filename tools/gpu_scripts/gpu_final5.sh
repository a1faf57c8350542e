cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f5_pytest.log 2>&1; tail -2 gpurun_out/f5_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f5_smoke.log 2>&1; tail -1 gpurun_out/f5_smoke.log
timeout 900 python bench.py > gpurun_out/f5_bench_1.log 2>&1; echo "bench1 rc=$?"
timeout 900 python bench.py --workload C4 > gpurun_out/f5_bench_C4.log 2>&1; echo "C4 rc=$?"
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 4 --master-port 29601 tools/check_fused.py C3 > gpurun_out/f5_check4.log 2>&1; echo "check4 rc=$?"; tail -2 gpurun_out/f5_check4.log
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port 2961$N bench.py --gpus $N > gpurun_out/f5_bench_$N.log 2>&1; echo "bench$N rc=$?"
done
for N in 1 2 4 C4; do grep '^{' gpurun_out/f5_bench_$N.log | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print(j['n_gpus'], j['ms_per_step'], j['value'], j['roofline']['frac'], {r:v['ms'] for r,v in j['per_rule'].items()}, j['clocks']['reasons'], j['e2e']['value'])"; done
