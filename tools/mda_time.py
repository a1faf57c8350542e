"""MDA per-call device time at the BASELINE configurations:
the whole call (Gram + D + enumeration of C(n, f) subsets + average) and the
selection from a ready Gram matrix alone."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth


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
for wl in (sys.argv[1:] or ["C1", "C2", "C3"]):
    cfg = synth.CONFIGS[wl]
    n, f, d = cfg.n, cfg.f, cfg.d
    X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
    a = gar.init("mda", n, f)
    out = torch.empty(d, device="cuda")
    ws = a.workspace(torch.device("cuda"))
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_gram_partial(X, G, ws, d=d)
    idx = torch.empty(64, dtype=torch.int32, device="cuda")
    res[wl] = {"n": n, "f": f, "d": d, "subsets": math.comb(n, f),
               "aggregate_ms": timed(lambda: a.aggregate(X, out=out, d=d)),
               "select_from_gram_ms": timed(lambda: gar.gar_select_from_gram("mda", G, n, f, 0, idx, workspace=ws)),
               "average_of_n_minus_f_ms": timed(lambda: gar.gar_combine("mda", X, f, 0, idx, out, d=d))}
    del X
    torch.cuda.empty_cache()
print(json.dumps(res))
