# Bulyan selection with register rows for n <= 64: GPU time (ncu launch list), parity suite
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/sel_launches.csv python tools/gram_vs_d2.py 47 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/sel_launches31.csv python tools/gram_vs_d2.py 31 > /dev/null 2>&1
python3 - <<'PY'
import csv, statistics
for fn in ("gpurun_out/sel_launches.csv", "gpurun_out/sel_launches31.csv"):
    rows = [r for r in csv.reader(open(fn)) if len(r) > 10]
    h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
    s = [float(r[vi].replace(",", "")) / 1000 for r in rows[1:] if "select_kernel" in r[ki]]
    print(fn, "select_kernel (Bulyan) median us", round(statistics.median(s), 2), len(s))
PY
timeout 1500 python -m pytest tests -m gpu -x -q > $o/sel_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $o/sel_pytest.log
timeout 600 python tools/sweep.py > $o/sel_sweep_f32.md 2>&1; echo "sweep rc=$?"; head -18 $o/sel_sweep_f32.md
