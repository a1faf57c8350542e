"""GPU parity for bf16 gradient inputs (R16): the
CUDA path through the ``_dt`` C entry points against the oracle applied to the
exactly-widened values (``oracle.widen_bf16``).  Same bar as the fp32 path:
bit-exact outputs and selections (exact on well-separated inputs), distances
within 1e-5 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import KRUM_FAMILY, assert_same_bits, assert_selection, distances_close

pytestmark = pytest.mark.gpu

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")


@pytest.fixture(scope="module")
def gar():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_05888_b200 as g
    return g


def to_device_bf16(bits: np.ndarray) -> torch.Tensor:
    """[n, d] uint16 bf16 patterns -> [n, ld] CUDA bf16 matrix, rows 16-byte aligned."""
    n, d = bits.shape
    ld = (d + 7) // 8 * 8
    B = np.zeros((n, ld), np.uint16)
    B[:, :d] = bits
    return torch.from_numpy(B.view(np.int16)).view(torch.bfloat16).cuda()


def recipe_bits(n, f, d, seed, kind="byzantine"):
    x = synth.make_gradients(n, f, d, seed=seed, ld=d, kind=kind)
    return synth.bf16_bits(synth.to_bf16(x))[:, :d]


def run(gar, rule, X, d, f, m=None):
    agg = gar.init(rule, X.shape[0], f, m)
    idx = torch.full((64,), -1, dtype=torch.int32, device=X.device)
    out = agg.aggregate(X, d=d, indices=idx if rule in KRUM_FAMILY or rule == "mda" else None)
    torch.cuda.synchronize()
    sel = idx[: agg.num_selected].cpu().numpy() if rule in KRUM_FAMILY or rule == "mda" else None
    return out.cpu().numpy(), sel


def check(gar, rule, bits, f, m=None, separated=False):
    n, d = bits.shape
    x = oracle.widen_bf16(bits)
    out, sel = run(gar, rule, to_device_bf16(bits), d, f, m)
    if rule in ("average", "median", "trimmed_mean"):
        assert_same_bits(out, oracle.aggregate(rule, x, f)[0], f"bf16 {rule}")
        return "exact"
    if rule == "mean_around_median":
        assert_same_bits(out, oracle.mean_around_median(x, f), "bf16 mean around median")
        return "exact"
    D = oracle.distances(x)
    mm = 1 if rule == "krum" else (n - f - 2 if m is None else m)
    verdict = assert_selection(rule, D, f, mm, sel, require_separated=separated)
    ref = oracle.bulyan_coordinate_phase(x, f, sel) if rule == "bulyan" else oracle.mean_of_rows(x, sel)
    assert_same_bits(out, ref, f"bf16 {rule} combine")
    return verdict


@pytest.mark.parametrize("n,f,d", [(11, 2, synth.MNIST_CNN_D), (19, 4, 200_003), (31, 7, 300_001),
                                   (7, 1, 4099), (63, 15, 40_005), (15, 3, 1), (5, 0, 9)])
@pytest.mark.parametrize("rule", RULES + ("mean_around_median",))
def test_bf16_recipe_parity(gar, rule, n, f, d):
    if rule == "bulyan" and n < 4 * f + 3:
        pytest.skip("quorum")
    check(gar, rule, recipe_bits(n, f, d, synth.BASE_SEED + 100 + n), f)


@pytest.mark.parametrize("n,f,d", [(11, 2, 79_510), (31, 7, 100_003), (64, 15, 12_001), (47, 11, 3001), (5, 0, 3001)])
@pytest.mark.parametrize("rule", KRUM_FAMILY)
def test_bf16_separated_selection_exact(gar, rule, n, f, d):
    """Well-separated bf16 inputs (d large enough that bf16 rounding keeps every
    decision gap above 1e-4; asserted): indices exactly the oracle's (on the
    widened values), combine bit-exact."""
    if rule == "bulyan" and n < 4 * f + 3:
        f = (n - 3) // 4
    bits = recipe_bits(n, f, d, synth.BASE_SEED + 9 * n, kind="separated")
    assert check(gar, rule, bits, f, separated=True) == "exact"


@pytest.mark.parametrize("n", list(range(1, 65)))
def test_bf16_every_n_coordinatewise(gar, n):
    """Every network size 1..64 on packed bf16x2 networks, tie-heavy columns,
    odd d (a pair straddles the end) and ragged tails."""
    rng = np.random.default_rng(4000 + n)
    d = 2 * 1000 + 2 * n + 1
    x = rng.standard_normal((n, d)).astype(np.float32)
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)
    bits[:, :60] = rng.choice(np.array([0x3F80, 0xBF80, 0x0000, 0x8000, 0x4000], np.uint16), (n, 60))
    f = (n - 1) // 2
    check(gar, "median", bits, f)
    for ft in sorted({0, f // 2, max(0, (n - 3) // 4), f}):
        check(gar, "trimmed_mean", bits, ft)
    check(gar, "average", bits, 0)
    check(gar, "mean_around_median", bits, max(0, (n - 3) // 4))


def test_bf16_adversarial_values(gar):
    """bf16 NaN (several payloads) / +-inf / -0 / subnormals / max finite."""
    specials = np.array([0x7FC0, 0xFFC1, 0x7F81, 0x7F80, 0xFF80, 0x8000, 0x0000, 0x0001, 0x8001, 0x7F7F, 0xFF7F],
                        np.uint16)
    for n, f in [(7, 1), (11, 2), (31, 7), (64, 15)]:
        rng = np.random.default_rng(n)
        d = 1037
        bits = ((rng.standard_normal((n, d)).astype(np.float32) * np.float32(0.01)).view(np.uint32) >> 16).astype(
            np.uint16)
        mask = rng.random((n, d)) < 0.08
        bits[mask] = rng.choice(specials, size=int(mask.sum()))
        bits[1] = bits[0]
        for rule in ("average", "median", "trimmed_mean", "mean_around_median"):
            check(gar, rule, bits, f if rule != "average" else 0)
        X = to_device_bf16(bits)
        x = oracle.widen_bf16(bits)
        for rule in KRUM_FAMILY:
            if rule == "bulyan" and n < 4 * f + 3:
                continue
            out, sel = run(gar, rule, X, d, f)
            ref = oracle.bulyan_coordinate_phase(x, f, sel) if rule == "bulyan" else oracle.mean_of_rows(x, sel)
            assert_same_bits(out, ref, f"bf16 {rule} adversarial")


@pytest.mark.parametrize("theta,f", [(3, 0), (5, 1), (7, 2), (9, 3), (12, 3), (17, 7), (33, 15), (64, 0)])
def test_bf16_bulyan_coordinate_phase_ties(gar, theta, f):
    """Integer-valued bf16 rows force closeness ties between different values
    (the exact rank-count path, per half of the bf16 pair)."""
    n = theta + 2 * f
    rng = np.random.default_rng(theta * 100 + f + 7)
    d = 2 * 1029 + 1
    x = rng.integers(-4, 5, (n, d)).astype(np.float32)
    x[:, ::7] = rng.standard_normal((n, len(range(0, d, 7)))).astype(np.float32)
    bits = (x.view(np.uint32) >> 16).astype(np.uint16)
    sel = rng.permutation(n)[:theta].astype(np.int32)
    out = torch.empty(d, dtype=torch.float32, device="cuda")
    gar.gar_combine_dt("bulyan", to_device_bf16(bits), f, 0, torch.from_numpy(sel).cuda(), out, d=d)
    torch.cuda.synchronize()
    assert_same_bits(out.cpu().numpy(), oracle.bulyan_coordinate_phase(oracle.widen_bf16(bits), f, sel),
                     "bf16 bulyan phase")


@pytest.mark.parametrize("n,d", [(3, 128), (8, 4093), (11, 79_511), (16, 20_000), (31, 300_001), (33, 50_001),
                                 (64, 100_003)])
def test_bf16_distances(gar, n, d):
    """gar_distances_dt (tensor-core Gram over the widened, centred rows)
    within 1e-5 of the oracle's fp64 distances, every NP instantiation."""
    bits = recipe_bits(n, max(0, (n - 3) // 4), d, 300 + n)
    ws = torch.empty(gar.gar_workspace_bytes("krum", n, 0, d), dtype=torch.uint8, device="cuda")
    Dg = torch.empty((n, n), dtype=torch.float64, device="cuda")
    gar.gar_distances_dt(to_device_bf16(bits), Dg, ws, d=d)
    torch.cuda.synchronize()
    distances_close(Dg.cpu().numpy(), oracle.distances(oracle.widen_bf16(bits)))


def test_bf16_gram_partial_and_combine_split(gar):
    """The d-sharded building blocks on bf16 rows: partial Grams of two
    coordinate slices sum to the Gram of the whole (selection identical), and
    gar_combine_dt on each slice reassembles the whole aggregate bit for bit."""
    n, f, d = 19, 4, 2 * 65_536 + 1000
    bits = recipe_bits(n, f, d, 77, kind="separated")
    X = to_device_bf16(bits)
    ws = torch.empty(gar.gar_workspace_bytes("bulyan", n, f, d), dtype=torch.uint8, device="cuda")
    h = 65_536
    G = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(2)]
    gar.gar_gram_partial_dt(X[:, :h], G[0], ws, d=h)
    gar.gar_gram_partial_dt(X[:, h:], G[1], ws, d=d - h)
    Gs = G[0] + G[1]
    for rule in KRUM_FAMILY:
        idx = torch.empty(64, dtype=torch.int32, device="cuda")
        k = gar.gar_select_from_gram(rule, Gs, n, f, 0, idx)
        whole, sel = run(gar, rule, X, d, f)
        assert list(idx[:k].cpu().numpy()) == list(sel)
        out = torch.empty(d, dtype=torch.float32, device="cuda")
        gar.gar_combine_dt(rule, X[:, :h], f, 0, idx, out[:h], d=h)
        gar.gar_combine_dt(rule, X[:, h:], f, 0, idx, out[h:], d=d - h)
        torch.cuda.synchronize()
        assert_same_bits(out.cpu().numpy(), whole, f"bf16 {rule} split combine")


def test_bf16_argument_checks(gar):
    """Misaligned bf16 rows (not 16-byte aligned) -> GAR_ERR_ALIGNMENT; an
    fp32 out overlapping a bf16 row -> GAR_ERR_INVALID_ARGUMENT; the fp32
    entry points still reject bf16 tensors."""
    from paper_2010_05888_b200._lib import GarError
    X = to_device_bf16(recipe_bits(7, 1, 1000, 5))
    with pytest.raises(GarError) as e:
        gar.gar_aggregate_dt("median", [X[i, 1:] for i in range(7)], 1, 0,
                             torch.empty(999, dtype=torch.float32, device="cuda"))
    assert e.value.code == 4
    with pytest.raises(TypeError):
        gar.gar_aggregate_ex("median", X, 1, 0, torch.empty(1000, dtype=torch.float32, device="cuda"), d=1000)
    flat = torch.zeros(8 * 1000, dtype=torch.bfloat16, device="cuda")
    rows = [flat[i * 1000:(i + 1) * 1000] for i in range(7)]
    out_alias = flat.view(torch.float32)[3000:4000]          # bytes [12000, 16000): row 6 is [12000, 14000)
    with pytest.raises(GarError) as e:
        gar.gar_aggregate_dt("median", rows, 1, 0, out_alias, d=1000)
    assert e.value.code == 1
