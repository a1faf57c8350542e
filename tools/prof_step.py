"""One step of the hot path on the C3 workload (n=31, f=7, d=25,557,032), for
ncu captures: warm-up step, then one profiled step (all six GARs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_2010_05888_b200 as gar

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
bf16 = len(sys.argv) > 2 and sys.argv[2] == "bf16"
cfg = synth.CONFIGS[wl] if not wl.startswith("sweep:") else synth.sweep_config(int(wl.split(":")[1]))
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
if bf16:
    X = synth.to_bf16(X)
aggs = {r: gar.init(r, n, f) for r in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")}
out = torch.empty(d, device="cuda")
for rep in range(2):
    for r, a in aggs.items():
        a.aggregate(X, out=out, d=d)
torch.cuda.synchronize()
print("ok")
