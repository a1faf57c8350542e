"""Per-call fixed cost of the Gram pass and the selection on the device: the
same calls eager and replayed from a CUDA graph (host overhead removed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

out = {}
for n in (19, 31, 47):
    for d in (131_072, 1_048_576, 6_389_258):
        f = (n - 3) // 4
        X = synth.make_gradients(n, f, d, seed=7, device="cuda")
        ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
        G = torch.empty((n, n), dtype=torch.float64, device="cuda")
        idx = torch.empty(64, dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()
        reps = 20

        def body():
            for _ in range(reps):
                gar.gar_gram_partial(X, G, ws, d=d, stream=s)

        def sel():
            for _ in range(reps):
                gar.gar_select_from_gram("bulyan", G, n, f, 0, idx, stream=s)
        with torch.cuda.stream(s):
            body(); sel()
        torch.cuda.synchronize()
        res = {}
        for name, fn in (("gram", body), ("select_bulyan", sel)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                fn()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            torch.cuda.synchronize()
            a.record(s)
            with torch.cuda.stream(s):
                fn()
            b.record(s)
            g.replay()
            c.record(s)
            torch.cuda.synchronize()
            res[name] = {"eager_us": round(a.elapsed_time(b) / reps * 1000, 1),
                         "graph_us": round(b.elapsed_time(c) / reps * 1000, 1)}
        out[f"n={n} d={d}"] = res
        del X
print(json.dumps(out))
