"""Both loaders of the coordinate-selection kernel (TMA bulk ring and direct
LDG) are exercised whatever the default policy picks: each
runs in a subprocess with GAR_COORD_LOADER forced, checked against the oracle.
The third case also turns off the compile-time-R Average for n <= 8, so the
general direct-load Average it replaces stays parity-tested."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import oracle, synth, paper_2010_05888_b200 as gar
from gpu_helpers import assert_same_bits, to_device
for n, f, d in [(7, 1, 5003), (31, 7, 70001), (33, 7, 9001), (63, 15, 30007), (64, 15, 1001)]:
    x = synth.make_gradients(n, f, d, seed=n, ld=d).numpy()
    x[:, :40] = np.random.default_rng(n).integers(-2, 3, (n, 40)).astype(np.float32)
    X = to_device(x)
    for rule in ("average", "median", "trimmed_mean"):
        out = gar.init(rule, n, f).aggregate(X, d=d).cpu().numpy()
        assert_same_bits(out, oracle.aggregate(rule, x, f)[0], rule)
    for rule in ("multi_krum", "bulyan"):
        idx = torch.full((64,), -1, dtype=torch.int32, device="cuda")
        agg = gar.init(rule, n, f)
        out = agg.aggregate(X, d=d, indices=idx).cpu().numpy()
        sel = idx[: agg.num_selected].cpu().numpy()
        ref = oracle.bulyan_coordinate_phase(x, f, sel) if rule == "bulyan" else oracle.mean_of_rows(x, sel)
        assert_same_bits(out, ref, rule)
print("ok")
"""


@pytest.mark.parametrize("loader", ["tma", "ldg", "ldg-general"])
def test_loader_forced(loader):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, GAR_COORD_LOADER=loader.split("-")[0])
    if loader == "ldg-general":
        env.update(GAR_AVG_RUNTIME_R="1")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
