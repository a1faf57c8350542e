#!/usr/bin/env python3
"""Summarise an ncu --set full report (and optionally a launch-list CSV) into
a markdown table + profiles/traffic.json (dram bytes per launch per kernel
class, read by bench.py's roofline.traffic).

    python tools/summarize_ncu.py gpurun_out/p22_full.ncu-rep [gpurun_out/p22_launches.csv] > profiles/r1_summary.md
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "time (us)",
    "dram__bytes_read.sum": "dram read",
    "dram__bytes_write.sum": "dram write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram %",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue %",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor %",
    "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed": "smem rd %",
    "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed": "smem wr %",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def kclass(name):
    if "gram_tc" in name:
        return "gram"
    if "coord_select" in name or "coord_ldg" in name or "copy_row" in name:
        return "coord_select"
    if "select_kernel" in name:
        return "select"
    if "gram_reduce" in name:
        return "gram_reduce"
    return "other"


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_us(val, unit):
    v = float(val.replace(",", ""))
    return v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)


def main(rep, launches=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    traffic = collections.defaultdict(list)
    per_kernel = collections.defaultdict(list)
    print(f"## ncu --set full: `{os.path.basename(rep)}`\n")
    print("| kernel | " + " | ".join(KEYS.values()) + " | top stalls |")
    print("|---" * (len(KEYS) + 2) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        cells = []
        for k in KEYS:
            if k not in d:
                cells.append("")
                continue
            if k == "gpu__time_duration.sum":
                cells.append(f"{to_us(d[k], u[k]):.1f}")
            elif k.startswith("dram__bytes"):
                cells.append(f"{to_bytes(d[k], u[k]) / 1e9:.3f} GB")
            else:
                cells.append(d[k])
        stalls = [(float(d[n].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                  for n in hdr if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")
                  and d.get(n)]
        tot = sum(s for s, _ in stalls) or 1
        top = ", ".join(f"{nm} {100 * s / tot:.0f}%" for s, nm in sorted(stalls, reverse=True)[:3])
        short = name.split("(")[0].replace("void ", "").replace("gar::", "").replace("<unnamed>::", "")
        print(f"| `{short}` | " + " | ".join(cells) + f" | {top} |")
        if "dram__bytes_read.sum" in d:
            b = (to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
                 + to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
            traffic[kclass(name)].append(b)
            per_kernel[short.split("<")[0]].append(b)
    summary = {k: int(sum(v) / len(v)) for k, v in traffic.items()}
    print("\nMean dram bytes (read + write) per launch, by kernel class: "
          + ", ".join(f"{k} {v / 1e9:.3f} GB" for k, v in summary.items()))
    if launches:
        print(f"\n## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`): `{os.path.basename(launches)}`\n")
        lr = list(csv.reader(open(launches)))
        start = next(i for i, r in enumerate(lr) if r and r[0] == "ID")
        h = lr[start]
        iname, ival, iunit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        per = collections.defaultdict(float)
        cnt = collections.defaultdict(int)
        total = 0.0
        for r in lr[start + 1:]:
            if len(r) <= ival:
                continue
            if kclass(r[iname]) == "other":
                continue
            nm = r[iname].split("(")[0].replace("void ", "").replace("gar::", "").replace("<unnamed>::", "")
            t = to_us(r[ival], r[iunit])
            per[nm] += t
            cnt[nm] += 1
            total += t
        print("| kernel | launches | total us | mean us per launch | share |\n|---|---|---|---|---|")
        for c, t in sorted(per.items(), key=lambda kv: -kv[1]):
            print(f"| `{c}` | {cnt[c]} | {t:.1f} | {t / cnt[c]:.1f} | {t / total:.3f} |")
    json.dump({"per_class": summary, "per_kernel": {k: int(sum(v) / len(v)) for k, v in per_kernel.items()},
               "source": os.path.basename(rep)},
              open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
