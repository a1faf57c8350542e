# executed SASS mix of the C3 coordinate kernels (trimmed mean, median, Bulyan phase, average) via ncu source counters
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'coord_select' \
  --launch-skip 4 -c 4 -o /tmp/mix -f python tools/prof_step.py C3 > $o/mix_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/mix.ncu-rep --page source --csv --print-source sass > /tmp/mix_src.csv 2>&1

python - <<'PY'
import csv
rows = list(csv.reader(open("/tmp/mix_src.csv")))
blocks, cur = [], None
for r in rows:
    if r and r[0] in ("Function Name", "Kernel Name"):
        cur = [r]; blocks.append(cur); continue
    if cur is not None: cur.append(r)
for i, b in enumerate(blocks):
    with open(f"/tmp/mix_{i}.csv", "w", newline="") as fh:
        csv.writer(fh).writerows(b[1:])
    print(i, b[0][1][:70] if len(b[0]) > 1 else "?", len(b))
PY
for i in 0 1 2 3; do echo "== kernel $i"; python tools/sass_mix.py /tmp/mix_$i.csv 25557032 | head -18; done > $o/mix_summary.txt 2>&1
cat $o/mix_summary.txt
