cd $GRAFT_REPO_ROOT
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29621 tools/check_fused.py C3 > gpurun_out/f9_check2.log 2>&1; echo "check2 rc=$?"
for N in 2 4; do
timeout 900 $R --nproc-per-node $N --master-port 2963$N bench.py --gpus $N > gpurun_out/f9_bench_$N.log 2>&1; echo "bench$N rc=$?"
timeout 900 $R --nproc-per-node $N --master-port 2964$N bench.py --gpus $N --workload C4 > gpurun_out/f9_bench_C4_$N.log 2>&1; echo "C4 bench$N rc=$?"
done
for f in f9_bench_2 f9_bench_4 f9_bench_C4_2 f9_bench_C4_4; do grep '^{' gpurun_out/$f.log | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('$f', j['n_gpus'], j['ms_per_step'], j['value'], {r:v['ms'] for r,v in j['per_rule'].items()}, j['clocks']['reasons'])"; done
