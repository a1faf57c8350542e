"""Does a fixed kernel slow down as the process runs?  Time the same call in
batches over ~20 s, and sample SM / memory clocks."""
import os, sys, json, subprocess, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth
cfg = synth.CONFIGS["C3"]
n, f, d = cfg.n, cfg.f, cfg.d
X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 2, device="cuda")
out = torch.empty(d, device="cuda")
aggs = {r: gar.init(r, n, f) for r in ("median", "krum", "bulyan")}
t_end = time.time() + float(sys.argv[1] if len(sys.argv) > 1 else 20)
while time.time() < t_end:
    row = {}
    for r, a in aggs.items():
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record()
        for _ in range(20):
            a.aggregate(X, out=out, d=d)
        e.record(); torch.cuda.synchronize()
        row[r] = round(s.elapsed_time(e) / 20, 4)
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw", "--format=csv,noheader"],
                       capture_output=True, text=True).stdout.strip()
    print(json.dumps(row), q, flush=True)
