"""Time one Gram pass (gar_gram_partial) at d = 25,557,032 for several n.
GAR_LIB_VARIANT selects an experiment build (tools/gram_exp.sh)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

bf16 = "--bf16" in sys.argv          # rows rounded to bf16 (gar_gram_partial_dt; 2 bytes per element)
ns = [int(a) for a in sys.argv[1:] if a != "--bf16"] or [15, 31, 47, 63]
d = synth.RESNET50_D
res = {}
for n in ns:
    X = synth.make_gradients(n, synth.sweep_config(n).f if n >= 7 else 0, d, seed=7, device="cuda")
    if bf16:
        X = synth.to_bf16(X)
    part = gar.gar_gram_partial_dt if bf16 else gar.gar_gram_partial
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for _ in range(3):
        part(X, G, ws, d=d)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(10):
        part(X, G, ws, d=d)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    res[n] = (round(ms, 4), round(n * d * (2 if bf16 else 4) / ms / 1e6 / 6533.5, 3))
    del X
    torch.cuda.empty_cache()
print(json.dumps({"variant": os.environ.get("GAR_LIB_VARIANT", "prod"), "bf16": bf16, "ms_frac": res}))
