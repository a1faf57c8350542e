"""Per-rule device times of one step on C3 (CUDA events), for A/B runs of tuning knobs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2010_05888_b200 as gar
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl] if not wl.startswith("sweep:") else synth.sweep_config(int(wl.split(":")[1]))
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
aggs = {r: gar.init(r, n, f) for r in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")}
out = torch.empty(d, device="cuda")
res = {}
for r, a in aggs.items():
    for _ in range(3):
        a.aggregate(X, out=out, d=d)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(10):
        a.aggregate(X, out=out, d=d)
    e.record(); torch.cuda.synchronize()
    res[r] = round(s.elapsed_time(e) / 10, 4)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("GAR_")}, "workload": wl, "ms": res}))
