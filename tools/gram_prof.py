"""Converter-warp cycle attribution (GRAM_EXP=5 build, libgar_exp5.so):
raw_full wait | loads+split | op_free wait | tcgen05.st+STS+wait::st | fences+arrive."""
import os, sys
os.environ["GAR_LIB_VARIANT"] = "exp5"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_05888_b200 as gar
import synth
d = synth.RESNET50_D
for n in [int(a) for a in sys.argv[1:]] or [7, 31, 63]:
    X = synth.make_gradients(n, 0, d, seed=7, device="cuda")
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    G = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_gram_partial(X, G, ws, d=d)
    gar.gar_gram_partial(X, G, ws, d=d)
    torch.cuda.synchronize()
    g = G.flatten()[:48].view(8, 6).cpu()
    tiles = g[:, 5]
    per = g[:, :5] / tiles[:, None]
    print(f"n={n} cycles per tile per converter warp (rawwait, load+split, opfree, st, fence+arrive):")
    for w in range(8):
        print("  warp", w, " ".join(f"{v:8.1f}" for v in per[w].tolist()), f" sum {per[w].sum():.0f}")
    del X
