"""Bulyan at C3 in three call contexts (device time, CUDA events): the single
C call (Aggregator.aggregate -> gar_aggregate_ex), the staged path bench.py
times (ShardedAggregator at world 1: Gram pass, select_from_gram, combine), and
the coordinate phase alone with the selected indices.  Rules are interleaved
as in one bench step when INTERLEAVE=1."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
from paper_2010_05888_b200.dist import ShardedAggregator
import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
out = torch.empty(d, device="cuda")
a1 = gar.init("bulyan", n, f)
a2 = ShardedAggregator("bulyan", n, f, d)
mk = gar.init("multi_krum", n, f)
idx = a1.select(X).clone()


def timed(fn, pre=None, reps=10):
    for _ in range(3):
        fn()
    ms = 0.0
    for _ in range(reps):
        if pre:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    return round(ms / reps, 4)


pre = (lambda: mk.aggregate(X, out=out, d=d)) if os.environ.get("INTERLEAVE") == "1" else None
res = {
    "aggregate_ex": timed(lambda: a1.aggregate(X, out=out, d=d), pre),
    "sharded_w1": timed(lambda: a2.aggregate(X, out_local=out), pre),
    "combine": timed(lambda: gar.gar_combine("bulyan", X, f, 0, idx, out, d=d), pre),
    "gram": timed(lambda: gar.gar_gram_partial(X, torch.empty((n, n), dtype=torch.float64, device="cuda"),
                                               torch.empty(gar.gar_workspace_bytes("bulyan", n, f, d), dtype=torch.uint8,
                                                           device="cuda"), d=d), pre),
}
print(json.dumps({"wl": wl, "env": {k: v for k, v in os.environ.items() if k.startswith(("GAR_", "INTER"))}, "ms": res}))
