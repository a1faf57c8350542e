"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the public Aggregator path on resident [n, d] matrices):

* C3 (ResNet-50-sized, n=31, f=7, d=25,557,032): every rule; coordinate-wise
  outputs checked on a sample of coordinates the oracle computes one by one;
  the Krum-family selections against the oracle's distance matrix over the
  whole vectors (exact or eps-tie), and their combine on the sample;
* C4 (VGG16-sized, n=31, f=7, d=138,357,544, 17 GB): Median on a sample, Krum
  with the oracle's distances accumulated over host-sized column chunks.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import KRUM_FAMILY, assert_same_bits, assert_selection, distances_close

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def gar():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_05888_b200 as g
    return g


def sample_columns(d, seed, k=1 << 16):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([np.arange(min(d, 4096)), np.arange(max(0, d - 4096), d),
                                    rng.integers(0, d, k)]))
    return idx


@pytest.fixture(scope="module")
def c3(gar):
    cfg = synth.CONFIGS["C3"]
    X = synth.make_gradients(cfg.n, cfg.f, cfg.d, seed=synth.BASE_SEED + 2, device="cuda")
    x = X[:, : cfg.d].cpu().numpy()
    D = oracle.distances(x)
    return cfg, X, x, D


@pytest.mark.parametrize("rule", ["average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"])
def test_c3_full_size(gar, c3, rule):
    cfg, X, x, D = c3
    n, f, d = cfg.n, cfg.f, cfg.d
    agg = gar.init(rule, n, f)
    idx = torch.full((64,), -1, dtype=torch.int32, device="cuda")
    out = agg.aggregate(X, d=d, indices=idx if rule in KRUM_FAMILY else None)
    torch.cuda.synchronize()
    cols = sample_columns(d, 3)
    got = out[torch.from_numpy(cols).cuda()].cpu().numpy()
    xs = np.ascontiguousarray(x[:, cols])
    if rule in KRUM_FAMILY:
        sel = idx[: agg.num_selected].cpu().numpy()
        mm = 1 if rule == "krum" else n - f - 2
        assert_selection(rule, D, f, mm, sel)
        ref = oracle.bulyan_coordinate_phase(xs, f, sel) if rule == "bulyan" else oracle.mean_of_rows(xs, sel)
    else:
        ref, _ = oracle.aggregate(rule, xs, f)
    assert_same_bits(got, ref, rule)


@pytest.fixture(scope="module")
def c3_separated(gar):
    cfg = synth.CONFIGS["C3"]
    X = synth.make_gradients(cfg.n, cfg.f, cfg.d, seed=synth.BASE_SEED + 12, device="cuda", kind="separated")
    x = X[:, : cfg.d].cpu().numpy()
    D = oracle.distances(x)
    yield cfg, X, x, D
    del X
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rule", KRUM_FAMILY)
def test_c3_full_size_separated_selection_exact(gar, c3_separated, rule):
    """At the full C3 size, in the launch configuration bench.py times, on an
    input whose oracle decisions are all separated by > 1e-4:
    the selected indices equal the oracle's exactly (distances over the whole
    25.6M-coordinate vectors), and the combine is bit-exact on a sample."""
    cfg, X, x, D = c3_separated
    n, f, d = cfg.n, cfg.f, cfg.d
    agg = gar.init(rule, n, f)
    idx = torch.full((64,), -1, dtype=torch.int32, device="cuda")
    out = agg.aggregate(X, d=d, indices=idx)
    torch.cuda.synchronize()
    sel = idx[: agg.num_selected].cpu().numpy()
    assert assert_selection(rule, D, f, 1 if rule == "krum" else n - f - 2, sel, require_separated=True) == "exact"
    cols = sample_columns(d, 5)
    xs = np.ascontiguousarray(x[:, cols])
    ref = oracle.bulyan_coordinate_phase(xs, f, sel) if rule == "bulyan" else oracle.mean_of_rows(xs, sel)
    assert_same_bits(out[torch.from_numpy(cols).cuda()].cpu().numpy(), ref, rule)


def test_c3_distances_full_size(gar, c3):
    cfg, X, x, D = c3
    ws = torch.empty(gar.gar_workspace_bytes("krum", cfg.n, 0, cfg.d), dtype=torch.uint8, device="cuda")
    Dg = torch.empty((cfg.n, cfg.n), dtype=torch.float64, device="cuda")
    gar.gar_distances(X, Dg, ws, d=cfg.d)
    torch.cuda.synchronize()
    distances_close(Dg.cpu().numpy(), D)


def test_c4_full_size_median_and_krum(gar):
    cfg = synth.CONFIGS["C4"]
    n, f, d = cfg.n, cfg.f, cfg.d
    X = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 3, device="cuda")
    cols = sample_columns(d, 4)
    tcols = torch.from_numpy(cols).cuda()
    xs = np.ascontiguousarray(X[:, tcols].cpu().numpy())
    out = gar.init("median", n, f).aggregate(X, d=d)
    assert_same_bits(out[tcols].cpu().numpy(), oracle.median(xs, f), "median C4")
    # Krum: oracle distances accumulated over column chunks (the definition's sum split by columns)
    D = np.zeros((n, n))
    chunk = 1 << 25
    for lo in range(0, d, chunk):
        hi = min(d, lo + chunk)
        D += oracle.distances(np.ascontiguousarray(X[:, lo:hi].cpu().numpy()))
    agg = gar.init("krum", n, f)
    idx = torch.full((64,), -1, dtype=torch.int32, device="cuda")
    out = agg.aggregate(X, d=d, indices=idx)
    sel = idx[:1].cpu().numpy()
    assert_selection("krum", D, f, 1, sel)
    assert_same_bits(out[tcols].cpu().numpy(), oracle.mean_of_rows(xs, sel), "krum C4")
    del X
    torch.cuda.empty_cache()
