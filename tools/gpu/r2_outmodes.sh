# N = 4: per-kernel times with each output mode (sharded / fused peer stores / multicast / NCCL all-gather)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
for m in sharded fused fused-mc replicated; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 20 --warmup 5 --output $m --e2e-steps 0 > $o/r2_out_$m.log 2>&1; echo "bench $m rc=$?"
done
python - <<'PY'
import json
for m in ("sharded", "fused", "fused-mc", "replicated"):
    ls = [l for l in open(f"gpurun_out/r2_out_{m}.log") if l.startswith("{")]
    if not ls: print(m, open(f"gpurun_out/r2_out_{m}.log").read()[-1500:]); continue
    j = json.loads(ls[0]); print(m, j["ms_per_step"], j["stages_ms"])
    for k, v in j["kernels"].items(): print(f"   {k:48s} {v['ms_per_launch']:.4f}")
PY
