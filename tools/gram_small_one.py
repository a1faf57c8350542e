"""ncu target: Gram pass + Bulyan selection at n = 31, d = 131072 (fixed costs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth

n, d = 31, 131_072
X = synth.make_gradients(n, 7, d, seed=7, device="cuda")
ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
G = torch.empty((n, n), dtype=torch.float64, device="cuda")
idx = torch.empty(64, dtype=torch.int32, device="cuda")
for _ in range(3):
    gar.gar_gram_partial(X, G, ws, d=d)
    gar.gar_select_from_gram("bulyan", G, n, 7, 0, idx)
torch.cuda.synchronize()
print("ok")
