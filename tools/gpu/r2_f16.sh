# 16-bit-operand Gram (gram_f16.cu): accuracy vs the oracle, time per pass against the tf32 kernel,
# then the parity suite and a bench line.
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 python tools/check_gram.py > $o/check_gram16.log 2>&1; echo "check_gram rc=$?"; cat $o/check_gram16.log
NS="15 17 19 23 31 32 33 35 47 63 64"
timeout 600 python tools/gram_time.py $NS 2>&1 | tail -1
GAR_GRAM=tf32 timeout 600 python tools/gram_time.py $NS 2>&1 | tail -1
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $o/pytest_all.log 2>&1; echo "all pytest rc=$?"; tail -12 $o/pytest_all.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $o/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
j = json.loads([l for l in open("gpurun_out/bench.log") if l.startswith("{")][0])
print("f32 ms/step", j["ms_per_step"], "value", j["value"], "roofline", j["roofline"]["kernel"], j["roofline"]["frac"])
for k, v in j["kernels"].items(): print(f"  {k:50s} {v['ms_per_launch']:.4f} ms frac {v['frac']}")
b = j["variants"]["bf16"]
print("bf16 ms/step", b["ms_per_step"], "value", b["value"])
for k, v in b["kernels"].items(): print(f"  {k:50s} {v['ms_per_launch']:.4f} ms frac {v['frac']}")
PY
