"""One Gram pass (gar_gram_partial) and one Median pass vs d at n = 31: the
fixed per-call cost a and per-coordinate cost b of t = a + b*d (tools only)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

n, f = 31, 7
res = {}
for d in (400_000, 800_000, 1_600_000, 3_200_000, 6_400_000, 12_800_000, 25_557_032):
    X = synth.make_gradients(n, f, d, seed=3, device="cuda")
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    out = torch.empty(d, device="cuda")
    med = gar.init("median", n, f)
    def t(fn):
        for _ in range(3): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(20): fn()
        b.record(); torch.cuda.synchronize()
        return round(a.elapsed_time(b) / 20 * 1000, 1)
    res[d] = {"gram_us": t(lambda: gar.gar_gram_partial(X, G, ws, d=d)), "median_us": t(lambda: med.aggregate(X, out=out, d=d))}
    del X
    torch.cuda.empty_cache()
print(json.dumps(res))
