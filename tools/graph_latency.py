"""Per-call latency of each GAR on a small configuration, eager (one C-ABI
call per aggregate) vs replaying a CUDA graph of the same call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

wl = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = synth.CONFIGS[wl]
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
res = {}
for r in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"):
    a = gar.init(r, n, f)
    out = torch.empty(d, device="cuda")
    ref = a.aggregate(X, out=torch.empty(d, device="cuda"), d=d).clone()
    replay = a.graphed(X, out, d=d)

    def timed(fn, reps=200):
        for _ in range(10):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(reps):
            fn()
        e.record(); torch.cuda.synchronize()
        return round(s.elapsed_time(e) / reps * 1000, 2)
    eager = timed(lambda: a.aggregate(X, out=out, d=d))
    graph = timed(replay)
    replay(); torch.cuda.synchronize()
    same = torch.equal(out.view(torch.int32), ref.view(torch.int32))
    res[r] = {"eager_us": eager, "graph_us": graph, "graph_output_bit_exact": same}
print(json.dumps({"workload": wl, "n": n, "f": f, "d": d, "per_call": res}))
