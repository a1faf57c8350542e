cd $GRAFT_REPO_ROOT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gvd_launches.csv python tools/gram_vs_d2.py 31 > /dev/null 2>&1; echo rc=$?
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/gvd_launches.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); gi = h.index("Grid Size")
seq = [(r[ki].split("(")[0][-40:], float(r[vi].replace(",", "")) / 1000, r[gi]) for r in rows[1:]]
# group consecutive runs of the same kernel
out = []
for k, v, g in seq:
    if out and out[-1][0] == k and out[-1][2] == g:
        out[-1][1].append(v)
    else:
        out.append([k, [v], g])
for k, v, g in out:
    v.sort()
    print(f"{len(v):3d} x median {v[len(v)//2]:8.2f} us grid {g:12s} {k}")
PY
