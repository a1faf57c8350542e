# final: clean-clone driver sequence on 1 GPU, then the scaling bench at N = 2 / 4 (default flags)
cd $GRAFT_REPO_ROOT
bash tools/clean_gpu_run.sh r2d > /dev/null 2>&1; tail -8 gpurun_out/clean_r2d.log | cut -c1-300
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/final_scale_$N.log 2>&1; echo "N=$N rc=$?"
done
for f in gpurun_out/clean_r2d.log gpurun_out/final_scale_2.log gpurun_out/final_scale_4.log; do python3 - $f <<'PY'
import json, sys
for line in open(sys.argv[1]):
    i = line.find('{"metric"')
    if i >= 0:
        j = json.loads(line[i:])
        rep = j.get("variants", {}).get("replicated_output", {})
        print(sys.argv[1], j["n_gpus"], j["value"], j["ms_per_step"], j["config"]["output"], "rep", rep.get("ms_per_step"),
              "roofline", j["roofline"]["kernel"], j["roofline"]["frac"], j["roofline"]["traffic"], "e2e", j["e2e"]["value"], j["clocks"])
PY
done
