"""Aggregate an ncu source page (--print-source cuda,sass CSV) by CUDA source line:
stall samples, instructions executed, shared wavefronts (+excessive).
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.defaultdict(lambda: [0, 0, 0, 0, collections.Counter(), ""])
fname, hdr = "?", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    d = dict(zip(hdr[2:], r[2:]))
    if not r[2]:
        continue
    key = (fname, r[0])
    a = agg[key]
    a[5] = r[1][:70]
    try:
        a[0] += int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
        a[1] += int(d.get("Instructions Executed", 0) or 0)
        a[2] += int(d.get("L1 Wavefronts Shared", 0) or 0)
        a[3] += int(d.get("L1 Wavefronts Shared Excessive", 0) or 0)
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k and v not in ("", "0"):
                a[4][k[6:]] += int(v)
    except ValueError:
        pass
tot = sum(a[0] for a in agg.values()) or 1
print(f"total samples {tot}")
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    st = ", ".join(f"{k} {v}" for k, v in a[4].most_common(3))
    print(f"{100*a[0]/tot:5.1f}% {a[1]:10d} inst  smem {a[2]:9d} (+{a[3]:8d})  {key[0]}:{key[1]:>4} {a[5]:70s} | {st}")
