# 4-GPU: oracle comparison of every sharded mode, then bench at N = 1, 2, 4 (fused output, the default)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
nvidia-smi -L
timeout 1200 python -m pytest tests/test_multigpu_gpu.py -q -x -p no:cacheprovider > $o/pytest_multi4.log 2>&1; echo "multi pytest rc=$?"; tail -3 $o/pytest_multi4.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-variants > $o/r2_bench_n1.log 2>&1; echo "bench N=1 rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N bench.py --gpus $N --steps 20 --warmup 5 > $o/r2_bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
done
python - <<'PY'
import json
for N in (1, 2, 4):
    f = f"gpurun_out/r2_bench_n{N}.log"
    ls = [l for l in open(f) if l.startswith("{")]
    if not ls: print(f, open(f).read()[-2000:]); continue
    j = json.loads(ls[0])
    print(N, "ms/step", j["ms_per_step"], "value", j["value"], "e2e", j["e2e"]["value"], j["config"]["output"], j["clocks"])
PY
