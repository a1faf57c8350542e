"""Fused server step: params <- params - lr * GAR(grads) with the
update in the producing kernel (gar_aggregate_sgd) vs aggregate + a separate
update (torch add_), per rule, at a workload.  Device time, CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
params = torch.randn(d, device="cuda")
out = torch.empty(d, device="cuda")
lr = 0.01


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
for r in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"):
    agg = gar.init(r, n, f)
    ws = agg.workspace(torch.device("cuda"))
    fused = timed(lambda: gar.gar_aggregate_sgd(r, X, f, 0, params, lr, workspace=ws, d=d))
    unfused = timed(lambda: (agg.aggregate(X, out=out, d=d), params.add_(out, alpha=-lr)))
    res[r] = {"fused_ms": fused, "aggregate_then_update_ms": unfused}
print(json.dumps({"workload": wl, "n": n, "f": f, "d": d, "per_rule": res}))
