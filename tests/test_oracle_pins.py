"""Pins for the CPU oracle (no GPU).  Each test fixes the oracle against
something other than itself: values the paper / SPEC prints, a hand-run worked
example, library routines (numpy, scipy), exact rational brute force, closed
forms and the invariants the paper states.  DESIGN.md §3 maps pin -> function.
"""
import itertools
import math

import numpy as np
import pytest
import scipy.spatial.distance as ssd
import scipy.stats

import oracle
from oracle import brute

RULES_QUORUM = {"median": 1, "trimmed_mean": 1, "krum": 3, "multi_krum": 3, "bulyan": 3}


def rnd(n, d, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((n, d)) * scale).astype(np.float32)


def planted(n, f, d, seed):
    """n-f honest rows near a common point, f far outliers."""
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal(d).astype(np.float32)
    x = (mu + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
    byz = rng.permutation(n)[:f]
    for t, b in enumerate(byz):
        x[b] = -100.0 * x[b] if t % 2 == 0 else rng.standard_normal(d).astype(np.float32) * 1e3
    honest = np.setdiff1d(np.arange(n), byz)
    return x, honest, byz


# --------------------------------------------------------------------------- SPEC examples
def test_spec_examples(golden):
    g = golden("spec_examples.json")
    for ex in g["average"]:
        np.testing.assert_array_equal(oracle.average(np.array(ex["x"], np.float32)), np.float32(ex["out"]))
    for ex in g["median"]:
        np.testing.assert_array_equal(oracle.median(np.array(ex["x"], np.float32), ex["f"]), np.float32(ex["out"]))
    mk = g["multi_krum"]
    x = np.tile(np.array(mk[0]["v"], np.float32), (mk[0]["copies"], 1))
    out, sel = oracle.multi_krum(x, mk[0]["f"], mk[0]["m"])
    np.testing.assert_array_equal(out, np.float32(mk[0]["out"]))
    assert list(sel) == [0, 1]                      # all scores 0 -> lowest indices (R5)
    x = np.array(mk[1]["x"], np.float32)
    out, sel = oracle.multi_krum(x, mk[1]["f"], mk[1]["m"])
    assert not set(mk[1]["never_selected"]) & set(sel.tolist())
    bu = g["bulyan"]
    x = np.tile(np.array(bu[0]["v"], np.float32), (bu[0]["copies"], 1))
    out, _ = oracle.bulyan(x, bu[0]["f"])
    np.testing.assert_array_equal(out, np.float32(bu[0]["out"]))
    out, _ = oracle.bulyan(np.array(bu[1]["x"], np.float32), bu[1]["f"])
    assert bu[1]["out_range"][0] <= out[0] <= bu[1]["out_range"][1]


def test_bulyan_worked_example(golden):
    g = golden("bulyan_worked_example.json")
    x = np.array(g["x"], np.float32).reshape(-1, 1)
    out, sel = oracle.bulyan(x, g["f"])
    assert sel.tolist() == g["selection"]
    assert out.view(np.uint32)[0] == int(g["out_bits_hex"], 16)
    # the brute force (exhaustive Krum rounds, rank-counting coordinate phase) agrees
    bout, bsel = brute.bulyan(x, g["f"])
    assert bsel.tolist() == g["selection"]
    assert bout.view(np.uint32)[0] == int(g["out_bits_hex"], 16)


def test_median3_formula_exhaustive(golden):
    """PAPER.md l.449-454 with floor division sorts every triple in {1,2,3}^3."""
    for v in itertools.product([1.0, 2.0, 3.0], repeat=3):
        assert list(oracle.median3_reorder(np.array(v, np.float32))) == sorted(v)
    for ex in golden("median3_formula.json")["examples"]:
        assert list(oracle.median3_reorder(np.array(ex["v"], np.float32))) == ex["w"]


# --------------------------------------------------------------------------- library routines
@pytest.mark.parametrize("n,d", [(1, 5), (7, 300), (31, 1000), (64, 257)])
def test_average_vs_numpy(n, d):
    x = rnd(n, d, n * 7 + d)
    ref = np.mean(x.astype(np.float64), axis=0).astype(np.float32)
    np.testing.assert_array_equal(oracle.average(x), ref)


@pytest.mark.parametrize("n,d", [(1, 3), (3, 100), (11, 500), (31, 1000), (63, 300)])
def test_median_vs_numpy_odd(n, d):
    x = rnd(n, d, n + d)
    np.testing.assert_array_equal(oracle.median(x, (n - 1) // 2), np.median(x, axis=0).astype(np.float32))


@pytest.mark.parametrize("n,d", [(2, 50), (10, 200), (64, 100)])
def test_median_vs_numpy_even(n, d):
    x = rnd(n, d, n + 3 * d)
    ref = np.median(x.astype(np.float64), axis=0).astype(np.float32)
    np.testing.assert_array_equal(oracle.median(x, 0), ref)


@pytest.mark.parametrize("n,f", [(3, 1), (11, 2), (19, 4), (31, 7), (63, 15), (20, 3), (44, 15)])
def test_trimmed_mean_vs_scipy(n, f):
    x = rnd(n, 400, n * f + 1)
    ref = scipy.stats.trim_mean(x.astype(np.float64), (f + 0.5) / n, axis=0).astype(np.float32)
    got = oracle.trimmed_mean(x, f)
    np.testing.assert_allclose(got, ref, rtol=2e-7, atol=1e-9)


def _round_f32(q):
    """Correctly rounded fp32 of an exact rational (ties to even)."""
    from fractions import Fraction
    lo = np.float32(float(q))
    while Fraction(float(lo)) > q:
        lo = np.nextafter(lo, np.float32(-np.inf))
    while Fraction(float(np.nextafter(lo, np.float32(np.inf)))) <= q:
        lo = np.nextafter(lo, np.float32(np.inf))
    hi = np.nextafter(lo, np.float32(np.inf))
    dl, dh = q - Fraction(float(lo)), Fraction(float(hi)) - q
    if dl < dh or (dl == dh and (int(lo.view(np.uint32)) & 1) == 0):
        return lo
    return hi


def test_sgd_update_pins():
    """The fused server step's update, fma(-lr, g, p): exact rational value
    rounded once to fp32; lr = 0 keeps p; p = g with lr = 1 gives 0."""
    from fractions import Fraction
    rng = np.random.default_rng(9)
    p = (rng.standard_normal(3000) * rng.choice([1e-3, 1.0, 1e3], 3000)).astype(np.float32)
    g = (rng.standard_normal(3000) * rng.choice([1e-4, 1.0, 1e4], 3000)).astype(np.float32)
    for lr in (np.float32(0.1), np.float32(1e-3), np.float32(3.0)):
        got = oracle.sgd_update(p, g, lr)
        for k in range(0, 3000, 7):
            exact = Fraction(float(p[k])) - Fraction(float(lr)) * Fraction(float(g[k]))
            assert got[k] == _round_f32(exact), (k, lr)
    np.testing.assert_array_equal(oracle.sgd_update(p, g, 0.0), p)
    assert np.all(oracle.sgd_update(g, g, 1.0) == 0)


def test_trimmed_membership_pins():
    """north_star: trimmed-set membership.  Pinned to rank counting (brute), to
    the kept count n - 2f, to f = 0 (everyone kept), and to the trimmed mean
    itself: the mean of the kept values in ascending order."""
    rng = np.random.default_rng(5)
    for n, f in [(1, 0), (5, 1), (7, 3), (11, 2), (31, 7), (64, 15)]:
        x = rng.integers(-3, 4, (n, 60)).astype(np.float32)       # many ties
        x[:, ::5] = rng.standard_normal((n, 12)).astype(np.float32)
        x[0, 3] = np.nan
        x[n - 1, 7] = -0.0
        mask = oracle.trimmed_membership(x, f)
        np.testing.assert_array_equal(mask, brute.trimmed_membership(x, f))
        counts = [bin(int(m)).count("1") for m in mask]
        assert counts == [n - 2 * f] * x.shape[1]
        tm = oracle.trimmed_mean(x, f)
        for k in range(x.shape[1]):
            kept = sorted(float(np.float32(np.inf) if np.isnan(x[i, k]) else x[i, k] + np.float32(0))
                          for i in range(n) if (int(mask[k]) >> i) & 1)
            s = 0.0
            for v in kept:
                s += v
            assert np.float32(s / len(kept)) == tm[k] or (np.isnan(tm[k]) and np.isnan(s))
    x = rng.standard_normal((9, 30)).astype(np.float32)
    assert np.all(oracle.trimmed_membership(x, 0) == np.uint64((1 << 9) - 1))


@pytest.mark.parametrize("n,d", [(3, 10), (11, 4099), (31, 9000)])
def test_distances_vs_scipy(n, d):
    x = rnd(n, d, n + d)
    D = oracle.distances(x)
    ref = ssd.cdist(x.astype(np.float64), x.astype(np.float64), "sqeuclidean")
    np.testing.assert_allclose(D, ref, rtol=1e-12, atol=0)
    assert np.all(np.diag(D) == 0) and np.array_equal(D, D.T)


def test_distances_closed_form():
    """x_i = i * 1 (constant rows)  =>  D_ij = (i - j)^2 * d exactly."""
    n, d = 9, 12345
    x = np.repeat(np.arange(n, dtype=np.float32)[:, None], d, axis=1)
    D = oracle.distances(x)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    np.testing.assert_array_equal(D, ((i - j) ** 2 * d).astype(np.float64))


def test_distances_nonfinite_and_overflow():
    x = rnd(5, 8, 1)
    x[2, 3] = np.nan
    x[4, 0] = np.inf
    D = oracle.distances(x)
    for r in (2, 4):
        assert np.all(np.isinf(np.delete(D[r], r)))
    assert np.isfinite(D[0, 1])
    y = np.zeros((3, 2), np.float32)
    y[0, 0] = 3e19                                      # square > FLT_MAX
    D = oracle.distances(y)
    assert D[0, 1] == math.inf and D[1, 2] == 0.0


# --------------------------------------------------------------------------- brute force, tiny inputs
def _tiny_cases(count, seed):
    rng = np.random.default_rng(seed)
    for _ in range(count):
        n = int(rng.integers(1, 10))
        d = int(rng.integers(1, 5))
        kind = rng.integers(0, 3)
        if kind == 0:
            x = rng.standard_normal((n, d)).astype(np.float32)
        elif kind == 1:     # many duplicates / ties
            x = rng.integers(-2, 3, (n, d)).astype(np.float32)
        else:               # specials
            x = rng.choice(np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 0.5], np.float32), (n, d))
        yield n, d, x


def test_coordinatewise_vs_brute():
    for n, d, x in _tiny_cases(600, 11):
        for f in range(0, (n - 1) // 2 + 1):
            np.testing.assert_array_equal(oracle.median(x, f), brute.median(x, f))
            np.testing.assert_array_equal(oracle.trimmed_mean(x, f), brute.trimmed_mean(x, f))
        np.testing.assert_array_equal(oracle.average(x), brute.average(x))


def test_distances_vs_exact_rational():
    for n, d, x in _tiny_cases(300, 12):
        np.testing.assert_allclose(oracle.distances(x), brute.distances(x), rtol=1e-15, atol=0)


def test_krum_family_vs_brute():
    rng = np.random.default_rng(13)
    checked = 0
    for _ in range(400):
        n = int(rng.integers(3, 10))
        d = int(rng.integers(1, 5))
        x = rng.standard_normal((n, d)).astype(np.float32)
        for f in range(0, (n - 3) // 2 + 1):
            D = oracle.distances(x)
            s = oracle.krum_scores(D, f)
            for m in range(1, n - f - 1):
                bsel, bs = brute.multi_krum_select(D, f, m)
                np.testing.assert_allclose(s, bs, rtol=1e-14, atol=0)
                assert oracle.multi_krum_select(D, f, m).tolist() == bsel.tolist()
                out, sel = oracle.multi_krum(x, f, m)
                np.testing.assert_array_equal(out, brute.mean_of_rows(x, bsel))
                checked += 1
            if n >= 4 * f + 3:
                bsel = brute.bulyan_select(D, f)
                assert oracle.bulyan_select(D, f).tolist() == bsel.tolist()
                np.testing.assert_array_equal(oracle.bulyan_coordinate_phase(x, f, bsel),
                                              brute.bulyan_coordinate_phase(x, f, bsel))
    assert checked > 500


def test_bulyan_round_scores_vs_brute():
    """oracle_bulyan_round_scores (the eps-tie replay function of the selection
    parity rule) against the brute-force subset minimum over
    random pools R: score_i = min over (|R|-f-2)-subsets of R\\{i} of the summed
    distances (reading R7), clamped at 0 neighbours; NaN
    outside the pool.  A wrong pool, n instead of |R|, or a missing clamp fails."""
    rng = np.random.default_rng(15)
    checked = 0
    for _ in range(300):
        n = int(rng.integers(2, 10))
        x = rng.standard_normal((n, int(rng.integers(1, 4)))).astype(np.float32)
        D = oracle.distances(x)
        for f in range(0, 3):
            pool = (rng.random(n) < 0.7).astype(np.uint8)
            if not pool.any():
                pool[int(rng.integers(0, n))] = 1
            members = [i for i in range(n) if pool[i]]
            k = max(len(members) - f - 2, 0)
            s = oracle.bulyan_round_scores(D, f, pool)
            for i in range(n):
                if not pool[i]:
                    assert np.isnan(s[i])
                    continue
                want = brute.krum_score(D, i, members, k)
                assert s[i] == pytest.approx(want, rel=1e-14, abs=0), (n, f, members, i)
                checked += 1
            # full pool: equals the Krum score table with n - f - 2 neighbours
            if n >= 2 * f + 3:
                np.testing.assert_allclose(oracle.bulyan_round_scores(D, f, np.ones(n, np.uint8)),
                                           oracle.krum_scores(D, f), rtol=0, atol=0)
    assert checked > 1000


def test_bulyan_coordinate_phase_ties_vs_brute():
    """Integer-valued inputs make closeness ties (equal |y - med| on both sides)."""
    rng = np.random.default_rng(14)
    for _ in range(300):
        f = int(rng.integers(0, 3))
        n = 4 * f + 3 + int(rng.integers(0, 3))
        x = rng.integers(-3, 4, (n, 3)).astype(np.float32)
        sel = rng.permutation(n)[: n - 2 * f].astype(np.int32)
        np.testing.assert_array_equal(oracle.bulyan_coordinate_phase(x, f, sel),
                                      brute.bulyan_coordinate_phase(x, f, sel))


# --------------------------------------------------------------------------- invariants from the paper
@pytest.mark.parametrize("rule", ["average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"])
def test_identical_inputs_return_the_input(rule):
    """north_star: identical honest inputs return that input (exact under R2)."""
    rng = np.random.default_rng(5)
    v = rng.standard_normal(777).astype(np.float32) * np.float32(3.3)
    for n in (7, 11, 31):
        f = (n - 3) // 4
        x = np.tile(v, (n, 1))
        out, _ = oracle.aggregate(rule, x, f)
        np.testing.assert_array_equal(out, v)


@pytest.mark.parametrize("n,f", [(7, 1), (11, 2), (19, 4), (31, 7)])
def test_range_confinement_planted_outliers(n, f):
    """with >= f+1 correct inputs, coordinate-wise Median is
    bounded by correct values; Bulyan / trimmed mean inherit the bound
    (SPEC.md l.115, l.540).  f outliers planted at random positions."""
    for seed in range(20):
        x, honest, _ = planted(n, f, 64, seed)
        lo, hi = x[honest].min(axis=0), x[honest].max(axis=0)
        for rule in ("median", "trimmed_mean", "bulyan"):
            out, _ = oracle.aggregate(rule, x, f)
            assert np.all(out >= lo) and np.all(out <= hi), rule


@pytest.mark.parametrize("n,f", [(7, 1), (11, 2), (31, 7)])
def test_krum_never_selects_planted_outliers(n, f):
    for seed in range(20):
        x, honest, byz = planted(n, f, 50, 100 + seed)
        _, sel = oracle.multi_krum(x, f)
        assert not set(sel.tolist()) & set(byz.tolist())
        # Bulyan round t uses max(n - t - f - 2, 0) neighbours; while that is
        # >= f an outlier's score contains an honest (far) distance, so rounds
        # 0 .. theta-2 are outlier-free.  The last round may degenerate (at
        # f = 1 it has 0 neighbours and the lowest index wins, reading R7).
        _, sel = oracle.bulyan(x, f)
        assert not set(sel[:-1].tolist()) & set(byz.tolist())


def test_median_order_statistic_property():
    """#{x < med} <= (n-1)/2 and #{x > med} <= (n-1)/2 and med is an input (odd n)."""
    for seed in range(30):
        n = 2 * (seed % 20) + 1
        x = rnd(n, 100, seed)
        med = oracle.median(x, 0)
        assert np.all((x < med).sum(0) <= (n - 1) // 2)
        assert np.all((x > med).sum(0) <= (n - 1) // 2)
        assert np.all((x == med).any(0))


def test_median_nan_is_plus_infinity():
    """R1: NaN orders as +inf, so f NaN rows act as outliers the median ignores."""
    x = rnd(7, 20, 3)
    x[[2, 5], :] = np.nan
    med = oracle.median(x, 2)
    y = x.copy()
    y[[2, 5], :] = np.inf
    np.testing.assert_array_equal(med, oracle.median(y, 2))
    assert np.all(np.isfinite(med))


def test_special_case_reductions():
    x = rnd(15, 333, 9)
    # trimmed mean f = 0 is the Average, n = 2f+1 is the Median (bit-exact)
    np.testing.assert_array_equal(oracle.trimmed_mean(x, 0), oracle.average(x))
    np.testing.assert_array_equal(oracle.trimmed_mean(x, 7), oracle.median(x, 7))
    # Bulyan with f = 0 keeps everything: theta = beta = n  ->  Average
    np.testing.assert_array_equal(oracle.bulyan(x, 0)[0], oracle.average(x))
    # Multi-Krum with m = 1 is Krum
    a, sa = oracle.multi_krum(x, 3, 1)
    b, sb = oracle.krum(x, 3)
    np.testing.assert_array_equal(a, b)
    assert sa.tolist() == sb.tolist()
    # n = 1: every coordinate-wise rule copies
    np.testing.assert_array_equal(oracle.median(x[:1], 0), x[0])


def test_permutation_equivariance():
    """Median/Average invariant under permutation; Krum-family
    selections permute with the inputs when scores are distinct."""
    x = rnd(11, 40, 21)
    perm = np.random.default_rng(1).permutation(11)
    for rule in ("average", "median", "trimmed_mean"):
        a, _ = oracle.aggregate(rule, x, 2)
        b, _ = oracle.aggregate(rule, x[perm], 2)
        if rule == "median":
            np.testing.assert_array_equal(a, b)
        else:
            np.testing.assert_allclose(a, b, rtol=1e-6)
    _, s = oracle.multi_krum(x, 2)
    _, sp = oracle.multi_krum(x[perm], 2)
    assert sorted(perm[sp].tolist()) == sorted(s.tolist())
    _, s, D = oracle.bulyan(x, 2, return_D=True)
    _, sp = oracle.bulyan(x[perm], 2)
    # compare rounds up to the first exact score tie (mutual nearest
    # neighbours tie when the neighbour count is 1; ties go by index, R5)
    pool = np.ones(11, np.uint8)
    for t, pick in enumerate(s):
        sc = oracle.bulyan_round_scores(D, 2, pool)
        best = np.nanmin(sc)
        if np.sum(sc == best) > 1:
            break
        assert perm[sp[t]] == pick
        pool[pick] = 0
    assert t >= 3


def test_translation_invariance_of_selection():
    x = rnd(19, 64, 31)
    _, s1 = oracle.bulyan(x, 4)
    _, s2 = oracle.bulyan(x + np.float32(0.5), 4)
    assert s1.tolist() == s2.tolist()


# --------------------------------------------------------------------------- preconditions
def test_quorum_preconditions(golden):
    golden("preconditions.json")
    x = rnd(10, 4, 0)
    with pytest.raises(oracle.OracleError) as e:
        oracle.median(x[:4], 2)             # 4 < 2*2+1
    assert e.value.code == oracle.QUORUM
    with pytest.raises(oracle.OracleError):
        oracle.trimmed_mean(x[:4], 2)
    with pytest.raises(oracle.OracleError) as e:
        oracle.multi_krum(x[:6], 2)         # 6 < 2*2+3
    assert e.value.code == oracle.QUORUM
    with pytest.raises(oracle.OracleError) as e:
        oracle.multi_krum(x, 2, 7)          # m > n - f - 2 = 6
    assert e.value.code == oracle.INVALID_M
    with pytest.raises(oracle.OracleError) as e:
        oracle.bulyan(x, 2)                 # 10 < 4*2+3
    assert e.value.code == oracle.QUORUM
    oracle.median(x[:5], 2)
    oracle.multi_krum(x[:7], 2)
    oracle.bulyan(x[:7], 1)


def test_thread_count_does_not_change_results():
    x = rnd(13, 50_001, 77)
    for fn in (lambda t: oracle.distances(x, t), lambda t: oracle.bulyan(x, 2, t)[0],
               lambda t: oracle.median(x, 3, t)):
        a, b = fn(1), fn(5)
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------- MDA
def test_mda_spec_example():
    """[(0), (1), (100)], f = 1 -> 0.5 (subset {0, 1}, diameter 1)."""
    out, sel = oracle.mda(np.array([[0.0], [1.0], [100.0]], np.float32), 1)
    assert out[0] == np.float32(0.5) and list(sel) == [0, 1]


def test_mda_vs_brute_force():
    """Subset enumeration with squared fp64 distances == itertools brute force
    with Euclidean (square-root, fsum) distances, on random small inputs."""
    rng = np.random.default_rng(21)
    for trial in range(40):
        n = int(rng.integers(1, 9))
        f = int(rng.integers(0, (n - 1) // 2 + 1))
        d = int(rng.integers(1, 5))
        x = rng.standard_normal((n, d)).astype(np.float32)
        out, sel = oracle.mda(x, f)
        bout, bsel = brute.mda(x, f)
        assert list(sel) == list(bsel), (n, f, sel, bsel)
        np.testing.assert_array_equal(out, bout)


def test_mda_special_cases_and_bounds():
    rng = np.random.default_rng(22)
    x = rng.standard_normal((9, 50)).astype(np.float32)
    np.testing.assert_array_equal(oracle.mda(x, 0)[0], oracle.average(x))         # f = 0: everyone
    v = rng.standard_normal(30).astype(np.float32)
    np.testing.assert_array_equal(oracle.mda(np.tile(v, (7, 1)), 3)[0], v)       # identical inputs
    with pytest.raises(oracle.OracleError):
        oracle.mda(x, 5)                                                          # q < 2f + 1
    # Lemma 1: with at most f Byzantine inputs, the output is within
    # the correct inputs' diameter of every correct input
    for trial in range(10):
        n, f = 11, 3
        h = (rng.standard_normal((n - f, 40)) * 0.1 + 1.0).astype(np.float32)
        byz = np.concatenate([-100 * h[:2], rng.standard_normal((1, 40)).astype(np.float32)])
        xs = np.concatenate([h, byz]).astype(np.float32)
        perm = rng.permutation(n)
        out, _ = oracle.mda(xs[perm], f)
        diam = max(np.linalg.norm(h[i].astype(np.float64) - h[j]) for i in range(n - f) for j in range(n - f))
        for i in range(n - f):
            assert np.linalg.norm(out.astype(np.float64) - h[i]) <= diam * (1 + 1e-6)
        # permutation invariance (no diameter ties with continuous inputs)
        out2, _ = oracle.mda(xs[rng.permutation(n)], f)
        np.testing.assert_allclose(out2, out, rtol=1e-6, atol=1e-7)


def test_mean_around_median_pins():
    """PAPER.md l.316 footnote: f = 0 keeps everyone (Average on finite data);
    n = 2f + 1 keeps only the median; range confinement with f planted
    outliers; a brute force (sort by closeness to the median, ties by index)."""
    rng = np.random.default_rng(31)
    x = rng.standard_normal((9, 300)).astype(np.float32)
    np.testing.assert_array_equal(oracle.mean_around_median(x, 0), oracle.average(x))   # exact fp64 sums
    np.testing.assert_array_equal(oracle.mean_around_median(x, 4), oracle.median(x, 4))
    h = (rng.standard_normal((8, 200)) * 0.1).astype(np.float32)
    xs = np.concatenate([h, 1e6 * np.ones((3, 200), np.float32)])
    out = oracle.mean_around_median(xs, 3)
    assert np.all(out >= h.min(axis=0)) and np.all(out <= h.max(axis=0))
    for k in range(0, 300, 37):
        col = x[:, k].astype(np.float64)
        med = np.median(col)
        order = sorted(range(9), key=lambda i: (abs(np.float32(col[i]) - np.float32(med)), i))[:9 - 2 * 2]
        kept = sorted(col[order])
        s = 0.0
        for v in kept:
            s += v
        assert np.float32(s / len(kept)) == oracle.mean_around_median(x, 2)[k]


def test_sanitize_spec_examples():
    """SPEC S:49-51."""
    nan, inf = np.nan, np.inf
    assert oracle.sanitize(np.array([[1, 2], [3, 4]], np.float32), 0) == ([0, 1], [])
    assert oracle.sanitize(np.array([[1, 2], [nan, 4], [5, 6]], np.float32), 1) == ([0, 2], [1])
    with pytest.raises(oracle.OracleError):
        oracle.sanitize(np.array([[nan, 1], [1, inf]], np.float32), 1)


# ---- bf16 inputs (R16) ------------------------------
# bf16 is the upper half of IEEE-754 binary32: sign, 8-bit exponent, 7 fraction
# bits.  These values follow from that definition alone.
BF16_GOLDEN = [
    (0x3F80, 1.0), (0xBF80, -1.0), (0x4000, 2.0), (0x4049, 3.140625), (0x3DCD, 0.10009765625),
    (0x0000, 0.0), (0x7F80, math.inf), (0xFF80, -math.inf),
    (0x0001, 2.0 ** -133),                 # smallest subnormal: 2^-126 * 2^-7
    (0x0080, 2.0 ** -126),                 # smallest normal
    (0x7F7F, (2.0 - 2.0 ** -7) * 2.0 ** 127),   # largest finite
    (0xC2C8, -100.0),
]


def test_widen_bf16_golden():
    bits = np.array([b for b, _ in BF16_GOLDEN], np.uint16)
    got = oracle.widen_bf16(bits)
    assert got.dtype == np.float32
    for (b, v), g in zip(BF16_GOLDEN, got):
        assert float(g) == v, hex(b)
    neg0 = oracle.widen_bf16(np.array([0x8000], np.uint16))[0]
    assert neg0 == 0.0 and math.copysign(1.0, float(neg0)) < 0
    assert np.isnan(oracle.widen_bf16(np.array([0x7FC0, 0xFFC1, 0x7F81], np.uint16))).all()


def test_widen_bf16_matches_torch_on_every_pattern():
    """All 65536 patterns against torch's own bfloat16 -> float32 conversion
    (an independent library routine)."""
    import torch
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ours = oracle.widen_bf16(bits)
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    same = (ours.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(ours) & np.isnan(ref))
    assert same.all()


def test_bf16_rules_are_the_fp32_rules_on_widened_values():
    """R16 end to end on a small case, against the brute forces: the median of
    bf16 inputs is itself a bf16 value (low 16 bits zero), and every rule
    equals the brute-force fp32 rule of the widened matrix."""
    rng = np.random.default_rng(15)
    n, f, d = 11, 2, 6
    x32 = (rng.standard_normal((n, d)) * 0.01).astype(np.float32)
    bits = (x32.view(np.uint32) >> 16).astype(np.uint16)           # truncation: any bf16 pattern will do
    bits[3, 2] = 0x7FC0                                             # a NaN payload
    bits[5, 4] = 0x8000                                             # -0
    xw = oracle.widen_bf16(bits)
    med = oracle.aggregate_bf16("median", bits, f)[0]
    assert (med.view(np.uint32) & 0xFFFF == 0).all()
    np.testing.assert_array_equal(med, np.array([brute.median(xw[:, k:k + 1], f)[0] for k in range(d)], np.float32))
    tm = oracle.aggregate_bf16("trimmed_mean", bits, f)[0]
    np.testing.assert_array_equal(tm, np.array([brute.trimmed_mean(xw[:, k:k + 1], f)[0] for k in range(d)],
                                               np.float32))
    out, sel = oracle.aggregate_bf16("bulyan", bits[:, [0, 1, 3, 5]], f)   # finite columns only
    bo, bs = brute.bulyan(xw[:, [0, 1, 3, 5]], f)
    np.testing.assert_array_equal(sel, bs)
    np.testing.assert_array_equal(out, bo)
