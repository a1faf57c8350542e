"""Executed-instruction mix by SASS opcode from an ncu source page
(ncu -i rep --page source --csv --print-source sass): thread-instructions per
opcode, and per unit of work if given (tools only).
    python tools/sass_mix.py page.csv [units]"""
import collections, csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr, mix = None, collections.Counter()
for r in rows:
    if r and "Source" in r and "Thread Instructions Executed" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    src = d.get("Source", "")
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(\.[A-Z0-9_]+)*)", src)
    if not m:
        continue
    try:
        t = float(d.get("Thread Instructions Executed", "0") or 0)
    except ValueError:
        continue
    mix[m.group(2).split(".")[0]] += t
tot = sum(mix.values())
print(f"total thread-instructions {tot:.4g}  per unit {tot / units:.1f}")
for op, t in mix.most_common(30):
    print(f"{op:14s} {t / units:9.2f}  {100 * t / tot:5.1f}%")
