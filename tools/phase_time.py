"""Time the Krum-family stages separately at C3: Gram pass, selection, combine
(Bulyan coordinate phase / Multi-Krum average / Krum copy)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl] if not wl.startswith("sweep:") else synth.sweep_config(int(wl.split(":")[1]))
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
out = torch.empty(d, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / reps, 4)


res = {}
ws = torch.empty(gar.gar_workspace_bytes("bulyan", n, f, d), dtype=torch.uint8, device="cuda")
G = torch.empty((n, n), dtype=torch.float64, device="cuda")
res["gram"] = timed(lambda: gar.gar_gram_partial(X, G, ws, d=d))
order = ("krum", "multi_krum", "bulyan") if os.environ.get("ORDER") != "rev" else ("bulyan", "multi_krum", "krum")
for rule in order:
    agg = gar.init(rule, n, f)
    idx = agg.select(X).clone()
    m = agg.m if hasattr(agg, "m") else 0
    res[f"combine_{rule}"] = timed(lambda: gar.gar_combine(rule, X, f, m, idx, out, d=d))
    res[f"select_from_gram_{rule}"] = timed(lambda: gar.gar_select_from_gram(rule, G, n, f, m, idx))
    res[f"select_{rule}"] = timed(lambda: agg.select(X))
    res[f"aggregate_{rule}"] = timed(lambda: agg.aggregate(X, out=out, d=d))

    def chain(rule=rule, m=m, idx=idx):
        gar.gar_gram_partial(X, G, ws, d=d)
        gar.gar_select_from_gram(rule, G, n, f, m, idx)
        gar.gar_combine(rule, X, f, m, idx, out, d=d)
    res[f"chain_{rule}"] = timed(chain)
print(json.dumps({"workload": wl, "env": {k: v for k, v in os.environ.items() if k.startswith("GAR_")}, "ms": res}))
