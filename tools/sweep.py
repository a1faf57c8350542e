"""BASELINE.json configs[4]: scaling sweep n in {7, 11, ..., 63}, f = (n-3)/4
(PAPER.md l.556), d = 25,557,032.  Per rule: device time (CUDA events, 10
calls after 3 warm-ups), gradient GB/s and fraction of the HBM roofline; plus
the Gram-vs-selection crossover: time of one Gram pass (gar_gram_partial)
against one coordinate-selection pass (Median) at each n.

    python tools/sweep.py > profiles/r1_sweep.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2010_05888_b200 as gar
import synth

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")
PEAK = 6533.5


def rule_bytes(rule, n, f, d, es=4):
    """rows read (es bytes per coordinate) + the fp32 output"""
    return es * d * {"average": n, "median": n, "trimmed_mean": n, "krum": n + 1,
                     "multi_krum": 2 * n - f - 2, "bulyan": 2 * n - 2 * f}[rule] + 4 * d


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    bf16 = "--bf16" in sys.argv
    es = 2 if bf16 else 4
    d = synth.RESNET50_D
    rows = []
    print("| n | f | " + " | ".join(f"{r} ms (HBM frac)" for r in RULES) + " | Gram pass ms | Median pass ms |")
    print("|---" * (len(RULES) + 4) + "|")
    for n in range(7, 64, 4):
        cfg = synth.sweep_config(n)
        f = cfg.f
        X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 5, device="cuda")
        if bf16:
            X = synth.to_bf16(X)
        out = torch.empty(d, device="cuda")
        res = {}
        for r in RULES:
            agg = gar.init(r, n, f)
            t = timed(lambda: agg.aggregate(X, out=out, d=d))
            res[r] = (t, rule_bytes(r, n, f, d, es) / (t * 1e-3) / 1e9 / PEAK)
        ws = torch.empty(gar.gar_workspace_bytes("krum", n, f, d), dtype=torch.uint8, device="cuda")
        G = torch.empty((n, n), dtype=torch.float64, device="cuda")
        tg = timed(lambda: (gar.gar_gram_partial_dt if bf16 else gar.gar_gram_partial)(X, G, ws, d=d))
        cells = " | ".join(f"{res[r][0]:.3f} ({res[r][1]:.2f})" for r in RULES)
        print(f"| {n} | {f} | {cells} | {tg:.3f} | {res['median'][0]:.3f} |", flush=True)
        rows.append({"n": n, "f": f, "ms": {r: res[r][0] for r in RULES}, "gram_ms": tg})
        del X
        torch.cuda.empty_cache()
    print("\n```json\n" + json.dumps(rows) + "\n```")


if __name__ == "__main__":
    main()
