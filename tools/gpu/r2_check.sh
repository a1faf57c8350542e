# full -m gpu suite + bench (f32 line with the bf16 variant)
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $o/pytest_all.log 2>&1; echo "all pytest rc=$?"; tail -6 $o/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
j = json.loads([l for l in open("gpurun_out/bench.log") if l.startswith("{")][0])
print("f32 ms/step", j["ms_per_step"], "value", j["value"], "roofline", j["roofline"]["kernel"], j["roofline"]["frac"], j["clocks"])
for k, v in j["kernels"].items(): print(f"  {k:50s} {v['ms_per_launch']:.4f} ms frac {v['frac']}")
b = j["variants"]["bf16"]
print("bf16 ms/step", b["ms_per_step"], "value", b["value"])
for k, v in b["kernels"].items(): print(f"  {k:50s} {v['ms_per_launch']:.4f} ms frac {v['frac']}")
PY
