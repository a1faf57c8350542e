"""The paper's GAR micro-benchmark protocol (Fig. 4a): d =
10^7, n = 7 upward, f = floor((n-3)/4), inputs resident in GPU memory, the
timing including the transfer of the result back to host memory, mean of 21
runs.  Reproduced on one B200 for context (the paper's only stated number:
Average ~ 8 ms on a GTX 1080 Ti, l.570)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

d = 10_000_000
rules = ("average", "median", "multi_krum", "mda", "bulyan")
rows = []
for n in (7, 11, 15, 19, 23, 27, 31):
    f = (n - 3) // 4
    X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 9, device="cuda")
    out = torch.empty(d, device="cuda")
    host = torch.empty(d, pin_memory=True)
    res = {}
    for r in rules:
        a = gar.init(r, n, f)
        for _ in range(3):
            a.aggregate(X, out=out, d=d)
            host.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(21):
            a.aggregate(X, out=out, d=d)
            host.copy_(out, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        res[r] = round(s.elapsed_time(e) / 21, 3)
    rows.append({"n": n, "f": f, "ms_incl_d2h": res})
    del X
    torch.cuda.empty_cache()
print(json.dumps(rows))
