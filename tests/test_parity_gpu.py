"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bar (north_star): bit-exact for Median,
trimmed mean, Average, the combine steps and selection indices (with the
eps-tie rule for near-ties); distances within 1e-5 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import (KRUM_FAMILY, assert_same_bits, assert_selection, distances_close, to_device)

pytestmark = pytest.mark.gpu

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")


@pytest.fixture(scope="module")
def gar():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_05888_b200 as g
    return g


def run_rule(gar, rule, X, d, f, m=None):
    agg = gar.init(rule, X.shape[0], f, m)
    idx = torch.full((64,), -1, dtype=torch.int32, device=X.device)
    out = agg.aggregate(X, d=d, indices=idx if rule in KRUM_FAMILY else None)
    torch.cuda.synchronize()
    sel = idx[: agg.num_selected].cpu().numpy() if rule in KRUM_FAMILY else None
    return out.cpu().numpy(), sel


def check_rule(gar, rule, x, f, m=None, X=None, separated=False):
    """separated: the input is synth kind="separated"; its selection must be exact."""
    n, d = x.shape
    X = to_device(x) if X is None else X
    out, sel = run_rule(gar, rule, X, d, f, m)
    if rule == "average":
        assert_same_bits(out, oracle.average(x), rule)
    elif rule == "median":
        assert_same_bits(out, oracle.median(x, f), rule)
    elif rule == "trimmed_mean":
        assert_same_bits(out, oracle.trimmed_mean(x, f), rule)
    else:
        D = oracle.distances(x)
        mm = 1 if rule == "krum" else (n - f - 2 if m is None else m)
        verdict = assert_selection(rule, D, f, mm, sel, require_separated=separated)
        if rule == "bulyan":
            assert_same_bits(out, oracle.bulyan_coordinate_phase(x, f, sel), rule)
        else:
            assert_same_bits(out, oracle.mean_of_rows(x, sel), rule)
        return verdict
    return "exact"


# ---------------------------------------------------------------- recipe inputs, several tiles + ragged tail
@pytest.mark.parametrize("n,f,d", [(11, 2, synth.MNIST_CNN_D), (19, 4, 200_003), (31, 7, 300_001),
                                   (7, 1, 4099), (63, 15, 40_005), (15, 3, 1)])
@pytest.mark.parametrize("rule", RULES)
def test_recipe_parity(gar, rule, n, f, d):
    x = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + n, ld=d).numpy()
    check_rule(gar, rule, x, f)


@pytest.mark.parametrize("n,f,d", [(11, 2, synth.MNIST_CNN_D), (19, 4, 200_003), (31, 7, 300_001),
                                   (7, 1, 4099), (63, 15, 40_005), (15, 3, 1), (64, 15, 3001), (47, 11, 3001),
                                   (5, 0, 3001), (4, 0, 1000)])
@pytest.mark.parametrize("rule", KRUM_FAMILY)
def test_separated_selection_exact(gar, rule, n, f, d):
    """Well-posed selections (every oracle decision gap > 1e-4, SURVEY.md
    §8c-6; asserted on the input): the GPU indices must equal the oracle's
    exactly, for Krum, Multi-Krum (default m and m = 3) and Bulyan (PAPER.md
    l.210-212, l.219-221), and the combine must be bit-exact."""
    if rule == "bulyan" and n < 4 * f + 3:
        f = (n - 3) // 4
    x = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 7 * n, ld=d, kind="separated").numpy()
    assert check_rule(gar, rule, x, f, separated=True) == "exact"
    if rule == "multi_krum" and n - f - 2 >= 3:
        assert check_rule(gar, rule, x, f, m=3, separated=True) == "exact"


@pytest.mark.parametrize("n", list(range(1, 65)))
def test_every_n_coordinatewise(gar, n):
    """Every network size 1..64 (odd and even n), including ragged d."""
    rng = np.random.default_rng(n)
    d = 1000 + 3 * n + 1
    x = rng.standard_normal((n, d)).astype(np.float32)
    x[:, :50] = rng.integers(-2, 3, (n, 50)).astype(np.float32)      # ties
    f = (n - 1) // 2
    check_rule(gar, "median", x, f)
    # the paper's f (n = 4f + 3, a pruned network) and other trims (full sort)
    for ft in sorted({0, f // 2, max(0, (n - 3) // 4), f}):
        check_rule(gar, "trimmed_mean", x, ft)
    check_rule(gar, "average", x, 0)


@pytest.mark.parametrize("n", [3, 5, 7, 8, 10, 11, 15, 19, 23, 31, 32, 33, 47, 63, 64])
def test_every_family_size(gar, n):
    f_b = (n - 3) // 4
    x = synth.make_gradients(n, f_b, 3001, seed=77 + n, ld=3001).numpy()
    check_rule(gar, "bulyan", x, f_b)
    f_k = (n - 3) // 2
    if f_k >= 0:
        check_rule(gar, "krum", x, f_k)
        check_rule(gar, "multi_krum", x, f_k)
        check_rule(gar, "multi_krum", x, f_k, m=1)


@pytest.mark.parametrize("theta,f", [(3, 0), (5, 1), (7, 1), (7, 2), (9, 2), (9, 3), (11, 4), (12, 3), (17, 7),
                                     (19, 8), (33, 15), (64, 0)])
def test_bulyan_coordinate_phase_ties(gar, theta, f):
    """Integer-valued rows force closeness ties between different values
    (exercises the exact rank-count path); the selection is given explicitly
    through gar_combine (n = theta + 2f rows)."""
    n = theta + 2 * f
    rng = np.random.default_rng(theta * 100 + f)
    d = 2053
    x = rng.integers(-4, 5, (n, d)).astype(np.float32)
    x[:, ::7] = rng.standard_normal((n, len(range(0, d, 7)))).astype(np.float32)
    sel = rng.permutation(n)[:theta].astype(np.int32)
    out = torch.empty(d, dtype=torch.float32, device="cuda")
    gar.gar_combine("bulyan", to_device(x), f, 0, torch.from_numpy(sel).cuda(), out, d=d)
    torch.cuda.synchronize()
    assert_same_bits(out.cpu().numpy(), oracle.bulyan_coordinate_phase(x, f, sel), "bulyan phase")


def test_adversarial_values(gar):
    """NaN / +-inf / -0 / 1e30 / denormals / duplicates / symmetric ties."""
    for n, f in [(7, 1), (11, 2), (31, 7), (64, 15)]:
        x = synth.adversarial_rows(n, 517, seed=n)
        for rule in ("average", "median", "trimmed_mean"):
            check_rule(gar, rule, x, f if rule != "average" else 0)
        # Krum family: non-finite rows get +inf distances; compare the combine given the GPU selection
        for rule in KRUM_FAMILY:
            if rule == "bulyan" and n < 4 * f + 3:
                continue
            X = to_device(x)
            out, sel = run_rule(gar, rule, X, x.shape[1], f)
            if rule == "bulyan":
                assert_same_bits(out, oracle.bulyan_coordinate_phase(x, f, sel), rule)
            else:
                assert_same_bits(out, oracle.mean_of_rows(x, sel), rule)


@pytest.mark.parametrize("n,f", [(1, 0), (5, 1), (7, 3), (11, 2), (19, 4), (31, 7), (33, 8), (64, 15), (64, 31)])
def test_trimmed_membership(gar, n, f):
    """north_star: trimmed-set membership bit-exact (gar_trimmed_membership vs
    the oracle), on tie-heavy and adversarial columns; and the product trimmed
    mean equals the ascending fp64 mean of the members the mask names."""
    rng = np.random.default_rng(1000 + n)
    d = 2 * 1031 + 3
    x = rng.integers(-3, 4, (n, d)).astype(np.float32)
    x[:, ::3] = rng.standard_normal((n, len(range(0, d, 3)))).astype(np.float32)
    x[:, -517:] = synth.adversarial_rows(n, 517, seed=n)
    X = to_device(x)
    mask = torch.empty(d, dtype=torch.int64, device="cuda")
    gar.gar_trimmed_membership(X, f, mask, d=d)
    out = torch.empty(d, dtype=torch.float32, device="cuda")
    gar.init("trimmed_mean", n, f).aggregate(X, out=out, d=d)
    torch.cuda.synchronize()
    got = mask.cpu().numpy().view(np.uint64)
    ref = oracle.trimmed_membership(x, f)
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, f"first mismatches at {bad[:5]}: {got[bad[:5]]} vs {ref[bad[:5]]}"
    res = out.cpu().numpy()
    canon = np.where(np.isnan(x), np.float32(np.inf), x + np.float32(0))
    for k in range(0, d, 97):
        kept = sorted(float(canon[i, k]) for i in range(n) if (int(got[k]) >> i) & 1)
        s = 0.0
        for v in kept:
            s += v
        assert_same_bits(np.float32(s / len(kept)).reshape(1), res[k:k + 1], f"trimmed mean at {k}")


@pytest.mark.parametrize("n,f,d", [(11, 2, 79_510), (31, 7, 300_001), (64, 15, 20_003)])
def test_fused_server_step(gar, n, f, d):
    """gar_aggregate_sgd: params <- fma(-lr, GAR(grads), params) inside the
    producing kernel equals the oracle's update applied to the (parity-tested)
    aggregate, bit for bit, for every rule; Krum family also via
    gar_combine_sgd on the selection."""
    x = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 17 + n, ld=d).numpy()
    X = to_device(x)
    rng = np.random.default_rng(n)
    p0 = rng.standard_normal(d).astype(np.float32)
    lr = np.float32(0.05)
    for rule in RULES:
        if rule == "bulyan" and n < 4 * f + 3:
            continue
        a = gar.init(rule, n, f)
        g = a.aggregate(X, out=torch.empty(d, dtype=torch.float32, device="cuda"), d=d)
        params = torch.from_numpy(p0.copy()).cuda()
        ws = a.workspace(torch.device("cuda"))
        gar.gar_aggregate_sgd(rule, X, f, 0, params, float(lr), workspace=ws, d=d)
        torch.cuda.synchronize()
        expect = oracle.sgd_update(p0, g.cpu().numpy(), lr)
        assert_same_bits(params.cpu().numpy(), expect, f"{rule} fused step")
        if rule in KRUM_FAMILY:
            idx = a.select(X, d=d)
            params2 = torch.from_numpy(p0.copy()).cuda()
            gar.gar_combine_sgd(rule, X, f, 0, idx, params2, float(lr), d=d)
            torch.cuda.synchronize()
            assert_same_bits(params2.cpu().numpy(), expect, f"{rule} fused combine step")


@pytest.mark.parametrize("n,f,d", [(1, 0, 100), (3, 1, 1000), (7, 2, 4099), (11, 2, 79_510), (15, 3, 20_003),
                                   (31, 7, 50_000), (64, 2, 3000)])
def test_mda_parity(gar, n, f, d):
    """MDA: the GPU's minimum-diameter subset equals the
    oracle's, or its diameter (oracle distances) is within 1e-5 of the
    minimum (eps-tie); the output equals the oracle's average of the GPU's
    subset bit for bit."""
    x = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 31 + n, ld=d).numpy() if n >= 3 else \
        np.random.default_rng(n).standard_normal((n, d)).astype(np.float32)
    X = to_device(x)
    a = gar.init("mda", n, f)
    out = a.aggregate(X, out=torch.empty(d, dtype=torch.float32, device="cuda"), d=d)
    sel = a.select(X, d=d).cpu().numpy()
    torch.cuda.synchronize()
    ref_out, ref_sel, D = oracle.mda(x, f, return_D=True)
    assert len(sel) == n - f and list(sel) == sorted(sel)

    def diam(s):
        return max((D[i, j] for i in s for j in s if i < j), default=0.0)
    if list(sel) != list(ref_sel):
        assert diam(sel) <= diam(ref_sel) * (1 + 1e-5), (sel, ref_sel, diam(sel), diam(ref_sel))
    assert_same_bits(out.cpu().numpy(), oracle.mean_of_rows(x, sel), "mda output")


def test_mda_special_inputs(gar):
    """SPEC S:89-91 ([(0), (1), (100)], f = 1 -> 0.5); identical inputs -> the
    lexicographically first subset and the input itself."""
    x = np.array([[0.0], [1.0], [100.0]], np.float32)
    out = gar.init("mda", 3, 1).aggregate(to_device(x), d=1)
    torch.cuda.synchronize()
    assert out.cpu().numpy()[0] == np.float32(0.5)
    v = np.random.default_rng(2).standard_normal(777).astype(np.float32)
    xs = np.tile(v, (9, 1))
    a = gar.init("mda", 9, 3)
    out = a.aggregate(to_device(xs), d=777)
    sel = a.select(to_device(xs), d=777).cpu().numpy()
    torch.cuda.synchronize()
    assert list(sel) == list(range(6))
    assert_same_bits(out.cpu().numpy(), v, "mda identical")


@pytest.mark.parametrize("n,f", [(1, 0), (4, 1), (7, 2), (11, 2), (12, 3), (31, 7), (31, 15), (64, 15)])
def test_mean_around_median_parity(gar, n, f):
    """Mean around median (PAPER.md l.316 footnote, R14) bit-exact against the
    oracle on recipe, tie-heavy and adversarial columns."""
    rng = np.random.default_rng(500 + n + f)
    d = 3 * 1031 + 1
    x = rng.standard_normal((n, d)).astype(np.float32)
    x[:, :400] = rng.integers(-2, 3, (n, 400)).astype(np.float32)
    x[:, -517:] = synth.adversarial_rows(n, 517, seed=n + f)
    out = gar.init("mean_around_median", n, f).aggregate(to_device(x), d=d)
    torch.cuda.synchronize()
    assert_same_bits(out.cpu().numpy(), oracle.mean_around_median(x, f), "mean around median")


GRAM_CC_MAX_N = 24   # csrc/gram.h kGramCckMaxN: the CUDA-core Gram up to it (and for 33..36), the tensor cores above


@pytest.mark.parametrize("n,d", [(7, 100_003), (15, 100_003), (19, 100_003), (31, 300_001), (35, 50_003), (64, 20_003)])
def test_gram_exchange_single_rank_and_staging(gar, n, d):
    """gar_gram_exchange with world = 1 (slots and flags in this GPU's memory):
    the flag handshake completes, G equals gar_gram_partial's bit for bit, and
    the staging copy (the fused ingress of the d-sharded path) equals the rows.
    The staging copy exists only in the tensor-core Gram, so for n <= 24 a
    staged exchange runs the other kernel than gar_gram_partial: equal there
    in D within the 1e-5 bar."""
    x = synth.make_gradients(n, (n - 3) // 4 if n >= 3 else 0, d, seed=5 + n, ld=d).numpy()
    X = to_device(x)
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    G0 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_gram_partial(X, G0, ws, d=d)
    slots = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    flags = torch.zeros(4, dtype=torch.int32, device="cuda")
    stage = torch.full((n, (d + 3) // 4 * 4), float("nan"), dtype=torch.float32, device="cuda")
    G1 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_gram_exchange(X, G1, ws, [slots.data_ptr()], [flags.data_ptr()], 0, 1, 1, d=d)
    torch.cuda.synchronize()
    assert torch.equal(G0, G1)
    for epoch in (2, 3):
        gar.gar_gram_exchange(X, G1, ws, [slots.data_ptr()], [flags.data_ptr()], 0, 1, epoch, d=d, stage=stage)
        torch.cuda.synchronize()
        if n > GRAM_CC_MAX_N and not 33 <= n <= 36:
            assert torch.equal(G0, G1), epoch
        else:   # G depends on each kernel's centring rows; D = G_ii + G_jj - 2 G_ij does not
            def dist(G):
                g = torch.diagonal(G)
                return g[:, None] + g[None, :] - 2 * G
            D0, D1 = dist(G0), dist(G1)
            off = ~torch.eye(n, dtype=torch.bool, device="cuda")
            assert float(((D0 - D1).abs()[off] / D0[off]).max()) <= 1e-5, epoch
    assert int(flags[0]) == 3
    assert torch.equal(stage[:, :d], X[:, :d])


def test_raw_address_rows(gar):
    """Rows given as raw device addresses (_lib.DevicePtrRows, the form the
    worker-major ingress uses for peer rows) aggregate exactly like the matrix."""
    from paper_2010_05888_b200._lib import DevicePtrRows
    n, f, d = 19, 4, 50_001
    X = to_device(synth.make_gradients(n, f, d, seed=8, ld=d).numpy())
    rows = DevicePtrRows([X.data_ptr() + i * X.stride(0) * 4 for i in range(n)], X.device)
    for rule in RULES:
        a = gar.init(rule, n, f)
        ref = a.aggregate(X, out=torch.empty(d, dtype=torch.float32, device="cuda"), d=d)
        got = a.aggregate(rows, out=torch.empty(d, dtype=torch.float32, device="cuda"), d=d)
        torch.cuda.synchronize()
        assert_same_bits(got.cpu().numpy(), ref.cpu().numpy(), rule)


@pytest.mark.parametrize("rule", ["median", "trimmed_mean", "multi_krum", "bulyan", "mda"])
def test_sanitize_and_aggregate(gar, rule):
    """SPEC S:43-51 on the GPU: gar_nonfinite_rows finds exactly the rows
    with a NaN / inf (SPEC examples included); aggregate_sanitized runs the rule
    on the rest with f reduced by their count, equal to the oracle's."""
    X = to_device(np.array([[1, 2], [np.nan, 4], [5, 6]], np.float32))
    assert gar.sanitize(X, 1, d=2) == ([0, 2], [1])
    with pytest.raises(gar.TooManyNonFinite):
        gar.sanitize(to_device(np.array([[np.nan, 1], [1, np.inf]], np.float32)), 1, d=2)
    n, f, d = 15, 3, 10_003
    x = synth.make_gradients(n, f, d, seed=41, ld=d).numpy()
    x[4, 77] = np.inf
    x[9, d - 1] = np.nan
    X = to_device(x)
    a = gar.init(rule, n, f)
    idx = torch.full((64,), -1, dtype=torch.int32, device="cuda")
    out, excluded = gar.aggregate_sanitized(a, X, d=d, indices=idx if rule != "median" and rule != "trimmed_mean"
                                            else None)
    torch.cuda.synchronize()
    kept, bad = oracle.sanitize(x, f)
    assert excluded == bad == [4, 9]
    xs, fs = np.ascontiguousarray(x[kept]), f - len(bad)
    got = out.cpu().numpy()
    if rule == "median":
        assert_same_bits(got, oracle.median(xs, fs), rule)
    elif rule == "trimmed_mean":
        assert_same_bits(got, oracle.trimmed_mean(xs, fs), rule)
    else:
        # selection (numbered among the kept rows) against the oracle, then a bit-exact combine
        ns = len(kept)
        D = oracle.distances(xs)
        if rule == "mda":
            sel = idx[: ns - fs].cpu().numpy()
            assert sel.tolist() == oracle.mda_select(D, fs).tolist()
            assert_same_bits(got, oracle.mean_of_rows(xs, sel), rule)
        elif rule == "multi_krum":
            sel = idx[: ns - fs - 2].cpu().numpy()
            assert_selection(rule, D, fs, ns - fs - 2, sel)
            assert_same_bits(got, oracle.mean_of_rows(xs, sel), rule)
        else:
            sel = idx[: ns - 2 * fs].cpu().numpy()
            assert_selection(rule, D, fs, 0, sel)
            assert_same_bits(got, oracle.bulyan_coordinate_phase(xs, fs, sel), rule)


def test_binding_rejects_bad_buffers(gar):
    """The binding checks what the C ABI cannot: dtype, device, size."""
    n, f, d = 7, 1, 1000
    X = torch.zeros((n, d), dtype=torch.float32, device="cuda")
    a = gar.init("median", n, f)
    with pytest.raises(TypeError):
        a.aggregate(X, out=torch.empty(d, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        a.aggregate(X, out=torch.empty(d - 1, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        a.aggregate(X, out=torch.empty(d, dtype=torch.float32))
    k = gar.init("multi_krum", n, f)
    ws = k.workspace(torch.device("cuda"))
    with pytest.raises(ValueError):          # room for fewer than m = n - f - 2 indices
        gar.gar_select("multi_krum", X, f, 0, torch.empty(2, dtype=torch.int32, device="cuda"), ws, d=d)
    with pytest.raises(ValueError):
        gar.gar_gram_partial(X, torch.empty(n * n - 1, dtype=torch.float64, device="cuda"), ws, d=d)


def test_graphed_aggregate_matches_eager(gar):
    """Aggregator.graphed: a CUDA graph of the call, replayed on new contents
    of the same buffers, equals the eager call bit for bit."""
    n, f, d = 11, 2, 79_510
    X = to_device(synth.make_gradients(n, f, d, seed=3, ld=d).numpy())
    for rule in RULES:
        a = gar.init(rule, n, f)
        out = torch.empty(d, dtype=torch.float32, device="cuda")
        replay = a.graphed(X, out, d=d)
        X.mul_(1.5).add_(0.25)                       # new contents, same addresses
        replay()
        ref = a.aggregate(X, out=torch.empty(d, dtype=torch.float32, device="cuda"), d=d)
        torch.cuda.synchronize()
        assert_same_bits(out.cpu().numpy(), ref.cpu().numpy(), rule)


def test_identical_inputs(gar):
    v = np.random.default_rng(3).standard_normal(10_007).astype(np.float32)
    for n in (7, 31, 63):
        f = (n - 3) // 4
        x = np.tile(v, (n, 1))
        for rule in RULES:
            out, _ = run_rule(gar, rule, to_device(x), x.shape[1], f)
            assert_same_bits(out, v, rule)


def test_distances_parity(gar):
    for n, f, d in [(11, 2, synth.MNIST_CNN_D), (31, 7, 250_001), (64, 15, 30_000), (2, 0, 17)]:
        x = synth.make_gradients(n, f, d, seed=5 + n, ld=d).numpy()
        X = to_device(x)
        ws = torch.empty(gar.gar_workspace_bytes("krum", max(n, 3), 0, d), dtype=torch.uint8, device="cuda")
        D = torch.empty((n, n), dtype=torch.float64, device="cuda")
        gar.gar_distances(X, D, ws, d=d)
        torch.cuda.synchronize()
        distances_close(D.cpu().numpy(), oracle.distances(x))


def _distances_within_norm_bound(D_gpu, x, D_ref, rel=1e-5):
    """The Gram method's error bound: fp32 products of centred rows, so the
    error of D_ij is relative to the centred squared norms, not to D_ij (with
    one coordinate, two nearly equal rows give a tiny D_ij by cancellation).
    Bound the kernel's centring row r* by the worst row: |x_i - c|^2 <=
    2 (|x_i - m|^2 + max_r |x_r - m|^2), m the coordinate-wise median."""
    xd = x.astype(np.float64)
    nrm = ((xd - np.median(xd, axis=0)) ** 2).sum(axis=1)
    scale = 2.0 * (nrm[:, None] + nrm[None, :] + 2.0 * nrm.max())
    err = np.abs(D_gpu - D_ref)
    assert np.all(err <= rel * (D_ref + scale)), f"max err / bound {np.max(err / (rel * (D_ref + scale) + 1e-300)):.3e}"


@pytest.mark.parametrize("n", list(range(2, 27)) + [32, 33, 34, 35, 36, 37])
def test_distances_every_small_n(gar, n):
    """Every n served by an exact-n CUDA-core Gram instantiation (n <= 15: all
    pairs per lane; 16..24: two pair chunks; 33..36: register blocks) and the
    tensor-core boundaries (25, 32, 37), at d values that leave ragged stages and tails (not multiples of
    the 1536 / 896 / 512-coordinate stages, nor of 4), fp32 rows and bf16 rows
    (widened exactly, R16).  d >= 4099: D within 1e-5 relative of the oracle;
    d = 1 (the global-load tail path only, where near-equal rows make D_ij a
    cancellation): within 1e-5 of the centred norms."""
    for d in (1, 4099, 30_011):
        x = synth.make_gradients(n, (n - 3) // 4 if n >= 3 else 0, d, seed=900 + n, ld=d).numpy()
        ws = torch.empty(gar.gar_workspace_bytes("krum", max(n, 3), 0, d), dtype=torch.uint8, device="cuda")
        D = torch.empty((n, n), dtype=torch.float64, device="cuda")
        xb = synth.to_bf16(torch.from_numpy(x))
        xw = oracle.widen_bf16(synth.bf16_bits(xb))[:, :d]
        for rows, ref_rows, call in ((to_device(x), x, gar.gar_distances), (xb.cuda(), xw, gar.gar_distances_dt)):
            call(rows, D, ws, d=d)
            torch.cuda.synchronize()
            Dg, Do = D.cpu().numpy(), oracle.distances(ref_rows)
            if d == 1:
                _distances_within_norm_bound(Dg, ref_rows, Do)
            else:
                distances_close(Dg, Do)


def test_distances_nonfinite(gar):
    x = np.random.default_rng(0).standard_normal((9, 1000)).astype(np.float32)
    x[3, 17] = np.nan
    x[6, 500] = np.inf
    ws = torch.empty(gar.gar_workspace_bytes("krum", 9, 0, 1000), dtype=torch.uint8, device="cuda")
    D = torch.empty((9, 9), dtype=torch.float64, device="cuda")
    gar.gar_distances(to_device(x), D, ws, d=1000)
    D = D.cpu().numpy()
    for r in (3, 6):
        assert np.all(np.isinf(np.delete(D[r], r)))
    distances_close(D, oracle.distances(x))


def test_sharded_building_blocks_equal_whole(gar):
    """gar_gram_partial over G coordinate slices, summed, then select + combine
    per slice == the single-call result (the d-sharded path)."""
    n, f, d = 31, 7, 100_000
    x = synth.make_gradients(n, f, d, seed=99, ld=d).numpy()
    X = to_device(x)
    for rule in KRUM_FAMILY:
        whole, sel = run_rule(gar, rule, X, d, f)
        ws = torch.empty(gar.gar_workspace_bytes(rule, n, f, d), dtype=torch.uint8, device="cuda")
        G = torch.zeros((n, n), dtype=torch.float64, device="cuda")
        bounds = [synth.shard_bounds(d, r, 4) for r in range(4)]
        parts = []
        for lo, hi in bounds:
            Gp = torch.empty((n, n), dtype=torch.float64, device="cuda")
            gar.gar_gram_partial([X[i, lo:hi] for i in range(n)], Gp, ws, d=hi - lo)
            parts.append(Gp)
        for Gp in parts:
            G += Gp
        idx = torch.empty(64, dtype=torch.int32, device="cuda")
        k = gar.gar_select_from_gram(rule, G, n, f, 0, idx)
        out = torch.empty(d, dtype=torch.float32, device="cuda")
        for lo, hi in bounds:
            gar.gar_combine(rule, [X[i, lo:hi] for i in range(n)], f, 0, idx, out[lo:hi], d=hi - lo)
        torch.cuda.synchronize()
        sel_sh = idx[:k].cpu().numpy()
        D = oracle.distances(x)
        mm = 1 if rule == "krum" else n - f - 2
        assert_selection(rule, D, f, mm, sel_sh)
        if sel_sh.tolist() == sel.tolist():
            assert_same_bits(out.cpu().numpy(), whole, rule)


def test_determinism(gar):
    x = synth.make_gradients(31, 7, 123_457, seed=4, ld=123_457).numpy()
    X = to_device(x)
    for rule in RULES:
        a, sa = run_rule(gar, rule, X, x.shape[1], 7)
        b, sb = run_rule(gar, rule, X, x.shape[1], 7)
        assert_same_bits(a, b, rule)
        if sa is not None:
            assert sa.tolist() == sb.tolist()


def test_empty_and_degenerate_sizes(gar):
    """d = 0 (nothing to aggregate: every rule succeeds and writes nothing;
    selections come from an all-zero distance matrix, i.e. index order),
    n = 1 (every coordinate-wise rule copies the row), d = 1 and d = 3 (all
    ragged, no bulk copy at all)."""
    n, f = 11, 2
    X = torch.zeros((n, 4), dtype=torch.float32, device="cuda")
    for rule in RULES:
        a = gar.init(rule, n, f)
        sentinel = torch.full((4,), 7.0, device="cuda")
        a.aggregate(X, out=sentinel, d=0)
        torch.cuda.synchronize()
        assert torch.all(sentinel == 7.0), rule
        if rule in KRUM_FAMILY:
            assert a.select(X, d=0).cpu().tolist() == list(range(a.num_selected)), rule
    v = np.random.default_rng(1).standard_normal((1, 1001)).astype(np.float32)
    for rule in ("average", "median", "trimmed_mean", "mean_around_median"):
        out = gar.init(rule, 1, 0).aggregate(to_device(v), d=1001)
        torch.cuda.synchronize()
        assert_same_bits(out.cpu().numpy(), v[0] + np.float32(0), rule)
    for d in (1, 3):
        x = np.random.default_rng(d).standard_normal((n, d)).astype(np.float32)
        for rule in RULES:
            check_rule(gar, rule, x, f)


def test_errors_from_python(gar):
    X = to_device(np.zeros((8, 16), np.float32))
    with pytest.raises(gar.GarError):
        gar.gar_aggregate_ex("median", X, 1, 0, X[0], d=16)               # out aliases row 0
    host = torch.zeros(16)
    with pytest.raises(gar.GarError) as e:
        # host pointer for out: rejected (no CPU fallback)
        import ctypes
        from paper_2010_05888_b200 import _lib
        arr, n, d, dev = _lib.row_pointers(X, 16)
        _lib.check(_lib.lib.gar_aggregate_ex(1, arr, n, 1, 0, 16, ctypes.c_void_p(host.data_ptr()), None, None, 0,
                                             None), "host out")
    assert e.value.code == 1


def test_interleaved_launch_configurations(gar):
    """One kernel launched with different shared-memory sizes in turn (Average
    over 31 rows, Multi-Krum's combine over 22, ...): the per-function
    dynamic shared-memory limit must never be left below a later launch's need."""
    n, f, d = 31, 7, 120_001
    x = synth.make_gradients(n, f, d, seed=123, ld=d).numpy()
    X = to_device(x)
    ref_avg = oracle.average(x)
    for _ in range(2):
        for rule in ("average", "multi_krum", "average", "bulyan", "trimmed_mean", "average", "krum", "median"):
            out, sel = run_rule(gar, rule, X, d, f)
            if rule == "average":
                assert_same_bits(out, ref_avg, rule)
