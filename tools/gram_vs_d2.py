"""Gram pass time vs d at fixed n (intercept = per-call fixed cost); also the
select kernel alone.  argv: n."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
res = {}
for d in (131_072, 1_048_576, 2_097_152, 4_194_304, 6_389_258):
    X = synth.make_gradients(n, (n - 3) // 4, d, seed=7, device="cuda")
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    idx = torch.empty(64, dtype=torch.int32, device="cuda")
    for _ in range(3):
        gar.gar_gram_partial(X, G, ws, d=d)
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize(); a.record()
    for _ in range(20):
        gar.gar_gram_partial(X, G, ws, d=d)
    b.record()
    for _ in range(20):
        gar.gar_select_from_gram("bulyan", G, n, (n - 3) // 4, 0, idx)
    c.record(); torch.cuda.synchronize()
    res[d] = {"gram_us": round(a.elapsed_time(b) / 20 * 1000, 1), "select_bulyan_us": round(b.elapsed_time(c) / 20 * 1000, 1)}
    del X
print(json.dumps({"n": n, "per_d": res}))
