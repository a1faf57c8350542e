"""ncu target: warm-up + one gar_gram_partial pass at d = 25,557,032 for n (argv[1])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
d = synth.RESNET50_D
X = synth.make_gradients(n, (n - 3) // 4 if n >= 3 else 0, d, seed=7, device="cuda")
ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
G = torch.empty((n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    gar.gar_gram_partial(X, G, ws, d=d)
torch.cuda.synchronize()
print("ok")
