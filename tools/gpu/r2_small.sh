# C1 / C2 per-call latency (eager vs graph) and the per-kernel device times of one Krum-family call
cd $GRAFT_REPO_ROOT
o=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $o/build.log 2>&1 || { tail -20 $o/build.log; exit 1; }
for wl in C1 C2; do timeout 300 python tools/graph_latency.py $wl 2>&1 | tail -1 | tee -a $o/small_latency.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/small_launches.csv python tools/graph_latency.py C1 > /dev/null 2>&1; echo "ncu rc=$?"
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/small_launches.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); v = v / 1000 if r[ui] == "nsecond" else v
    agg[r[ki].split("(")[0][:70]].append(v)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    v.sort(); print(f"{len(v):5d} x  median {v[len(v)//2]:8.2f} us  {k}")
PY
