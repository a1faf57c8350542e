# min/max pipe microbenchmark + bf16 re-bench after the O(theta) Bulyan tie path.
cd $GRAFT_REPO_ROOT
o=gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipebench tools/pipebench.cu && /tmp/pipebench > $o/pipebench.log 2>&1; cat $o/pipebench.log
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 900 python -m pytest tests/test_bf16_gpu.py -q -x -p no:cacheprovider > $o/pytest_bf16.log 2>&1; echo "bf16 pytest rc=$?"; tail -3 $o/pytest_bf16.log
timeout 600 python bench.py --steps 10 --warmup 3 --dtype bf16 --no-cpu-baseline > $o/bench_bf16.log 2>&1; echo "bench bf16 rc=$?"
python - <<'PY'
import json
j = json.loads([l for l in open("gpurun_out/bench_bf16.log") if l.startswith("{")][0])
print("bf16 ms/step", j["ms_per_step"], "value", j["value"])
for k, v in j["kernels"].items(): print(f"  {k:50s} {v['ms_per_launch']:.4f} ms frac {v['frac']}")
PY
