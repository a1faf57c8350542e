# centre-pick padding: Gram fixed cost (ncu launch list vs d), accuracy, parity subset
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
bash tools/gpu/r2_gram_fixed.sh
python3 - <<'PY'
import csv, statistics
rows = [r for r in csv.reader(open("gpurun_out/gvd_launches.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
g = [float(r[vi].replace(",", "")) / 1000 for r in rows[1:] if "gram_tc" in r[ki]]
for i in range(5):
    print("d index", i, "gram_tc median us", round(statistics.median(g[i*23:(i+1)*23]), 2))
PY
timeout 600 python tools/check_gram.py 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q -k "gram or distances or krum or bulyan or selection or family" > gpurun_out/pick_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pick_pytest.log
timeout 300 python tools/gram_time.py 31 35 63 2>&1 | tail -1
