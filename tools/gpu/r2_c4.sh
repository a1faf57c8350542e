# C4 (VGG16-sized, d = 138M, n = 31) bench at N = 1 / 2 / 4, default flags (sharded output at N > 1)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c4_1.log 2>&1; echo "N=1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 \
    bench.py --gpus $N --workload C4 --steps 10 --warmup 3 > gpurun_out/c4_$N.log 2>&1; echo "N=$N rc=$?"
done
for N in 1 2 4; do python3 - $N <<'PY'
import json, sys
for line in open(f"gpurun_out/c4_{sys.argv[1]}.log"):
    if line.startswith('{"metric"'):
        j = json.loads(line)
        rep = j.get("variants", {}).get("replicated_output", {})
        print(sys.argv[1], j["value"], j["ms_per_step"], j["config"]["output"], "rep", rep.get("ms_per_step"),
              {k: v["ms"] for k, v in j["per_rule"].items()}, j["clocks"])
PY
done
