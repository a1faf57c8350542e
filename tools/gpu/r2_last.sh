# last check of the round: smoke, full GPU suite, reference arm, default bench
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/last_pytest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/last_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/last_ref.log
timeout 900 python bench.py > gpurun_out/last_bench.log 2>&1; echo "bench rc=$?"
python3 - <<'PY'
import json
for line in open("gpurun_out/last_bench.log"):
    if line.startswith('{"metric"'):
        j = json.loads(line)
        print(j["value"], j["ms_per_step"], j["roofline"]["kernel"], j["roofline"]["frac"], j["roofline"]["traffic"], j["gpu_launches"], j["clocks"])
        print({k: (v["ms"], v["roofline_frac"]) for k, v in j["per_rule"].items()})
PY
