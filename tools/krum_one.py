"""ncu target: warm-up + one Krum-family aggregate at a small configuration (argv: workload rule)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C2"
rule = sys.argv[2] if len(sys.argv) > 2 else "krum"
cfg = synth.CONFIGS[wl]
X = synth.make_gradients(cfg.n, cfg.f, cfg.d, seed=synth.BASE_SEED + 2, device="cuda")
a = gar.init(rule, cfg.n, cfg.f)
out = torch.empty(cfg.d, device="cuda")
for _ in range(4):
    a.aggregate(X, out=out, d=cfg.d)
torch.cuda.synchronize()
print("ok")
