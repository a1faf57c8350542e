"""Quick GPU check of the tensor-core Gram: gar_distances vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2010_05888_b200 as gar

def run(x):
    n, d = x.shape
    X = torch.zeros((n, (d + 3) // 4 * 4), dtype=torch.float32)
    X[:, :d] = torch.from_numpy(x)
    X = X.cuda()
    ws = torch.empty(gar.gar_workspace_bytes("krum", max(n, 3), 0, d), dtype=torch.uint8, device="cuda")
    D = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_distances(X, D, ws, d=d)
    torch.cuda.synchronize()
    return D.cpu().numpy()

for (n, f, d, kind) in [(3, 0, 128, "clean"), (5, 1, 1000, "byzantine"), (7, 1, 300001, "byzantine"),
                        (8, 1, 4093, "clean"), (10, 1, 77777, "byzantine"), (11, 2, 79510, "byzantine"), (12, 2, 250001, "clean"), (13, 2, 99999, "byzantine"), (15, 3, 333333, "clean"), (16, 3, 77777, "clean"), (17, 3, 5000, "byzantine"), (22, 4, 222222, "byzantine"),
                        (19, 4, 1756426, "byzantine"), (23, 5, 123457, "clean"),
                        (31, 7, 300001, "byzantine"), (32, 7, 4096, "clean"), (33, 7, 50000, "byzantine"),
                        (64, 15, 100003, "byzantine")]:
    x = synth.make_gradients(n, f, d, seed=1 + n, ld=d, kind=kind).numpy()
    t = time.time()
    Dg = run(x)
    Do = oracle.distances(x)
    m = Do > 0
    rel = np.abs(Dg - Do)[m] / Do[m]
    print(f"n={n} d={d} {kind}: max rel err {rel.max():.3e} median {np.median(rel):.3e}  diag0 {np.abs(np.diag(Dg)).max()}", flush=True)
# high-similarity honest gradients: large common mean, tiny spread
rng = np.random.default_rng(0)
mu = rng.standard_normal(200000).astype(np.float32)
x = (mu + 1e-3 * rng.standard_normal((31, 200000))).astype(np.float32)
Dg, Do = run(x), oracle.distances(x)
m = Do > 0
print("high-similarity (cos~0.999999): max rel err", (np.abs(Dg - Do)[m] / Do[m]).max())
