"""GPU check of the Gram on bf16 rows: gar_distances_dt vs the fp64 oracle on
the exactly widened values (R16), n spanning the CUDA-core (<= 22)
and tensor-core (bf16 hi/lo operands, kind::f16) kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2010_05888_b200 as gar


def run(xb):
    n = xb.shape[0]
    X = xb.cuda()
    d = X.shape[1]
    ws = torch.empty(gar.gar_workspace_bytes("krum", max(n, 3), 0, d), dtype=torch.uint8, device="cuda")
    D = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_distances_dt(X, D, ws, d=d)
    torch.cuda.synchronize()
    return D.cpu().numpy()


def check(x, label):
    xb = synth.to_bf16(torch.from_numpy(x))
    Dg = run(xb)
    Do = oracle.distances(oracle.widen_bf16(synth.bf16_bits(xb)))
    m = Do > 0
    rel = np.abs(Dg - Do)[m] / Do[m]
    print(f"{label}: max rel err {rel.max():.3e} median {np.median(rel):.3e}", flush=True)
    return rel.max()


worst = 0.0
for (n, f, d, kind) in [(19, 4, 300_001, "byzantine"), (23, 5, 123_457, "clean"), (31, 7, 300_001, "byzantine"),
                        (32, 7, 4096, "clean"), (33, 7, 50_000, "byzantine"), (47, 11, 100_003, "byzantine"),
                        (64, 15, 100_003, "byzantine")]:
    x = synth.make_gradients(n, f, d, seed=1 + n, ld=d, kind=kind).numpy()
    worst = max(worst, check(x, f"n={n} d={d} {kind}"))
rng = np.random.default_rng(0)
mu = rng.standard_normal(200_000).astype(np.float32)
for n in (19, 31, 47):
    x = (mu + 1e-2 * rng.standard_normal((n, 200_000))).astype(np.float32)
    worst = max(worst, check(x, f"high-similarity n={n} (spread 1e-2)"))
# magnitudes spanning many binades per coordinate (exponent gaps > 7 vs the centre)
x = (rng.standard_normal((31, 100_000)) * np.exp(rng.uniform(-12, 12, (31, 100_000)))).astype(np.float32)
worst = max(worst, check(x, "n=31 log-uniform magnitudes (e^-12..e^12)"))
print("worst", worst)
