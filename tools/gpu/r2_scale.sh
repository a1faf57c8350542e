# C3 bench at N = 1 / 2 / 4 (default: sharded output, replicated variant), as the driver launches it
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 python bench.py --steps 20 --warmup 5 > $o/scale_1.log 2>&1; echo "N=1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus $N --steps 20 --warmup 5 > $o/scale_$N.log 2>&1; echo "N=$N rc=$?"
done
for N in 1 2 4; do python3 - $N <<'PY'
import json, sys
N = sys.argv[1]
for line in open(f"gpurun_out/scale_{N}.log"):
    if line.startswith('{"metric"'):
        j = json.loads(line)
        rep = j.get("variants", {}).get("replicated_output", {})
        print(N, j["value"], j["ms_per_step"], j["config"]["output"], "replicated:", rep.get("ms_per_step"), rep.get("value"),
              "e2e", j["e2e"]["value"], "clocks", j["clocks"])
PY
done
