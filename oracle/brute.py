"""Independent pure-Python brute forces (tiny inputs only) that PIN the oracle.

TEST INFRASTRUCTURE ONLY.  Each function computes the same quantity as the C++
oracle by a *different* method, so that a dropped term, a wrong sign/index or a
transposed operand in either shows up as a mismatch:

* median       — order-statistic definition by counting (no sorting);
* trimmed mean — repeated removal of the current min and max, exact fsum;
* distances    — exact rational arithmetic (fractions.Fraction);
* Krum score   — minimum over ALL neighbour subsets of the prescribed size
                 (itertools.combinations), instead of "sum of the smallest";
* Bulyan       — literal replay of the rounds with exhaustive Krum, and the
                 coordinate phase by rank counting instead of sorting.

Readings R1-R9 are the ones of DESIGN.md §3.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np


def _canon(v: float) -> float:
    v = float(v)
    if math.isnan(v):
        return math.inf
    if v == 0.0:
        return 0.0
    return v


def _f32(v: float) -> float:
    return float(np.float32(v))


def _mean_f32(vals) -> float:
    """fp32 rounding of (exactly rounded sum) / count, via fp64 like R2.
    For non-finite values fall back to plain float arithmetic."""
    vals = [float(v) for v in vals]
    if all(math.isfinite(v) for v in vals):
        s = math.fsum(vals)
    else:
        s = sum(vals)
    return _f32(s / len(vals))


def median(x, f=0):
    x = np.asarray(x, np.float32)
    n, d = x.shape
    out = np.empty(d, np.float32)
    for k in range(d):
        c = [_canon(x[i, k]) for i in range(n)]
        h = (n - 1) // 2
        # order statistic of rank h: the value v with #{<v} <= h < #{<=v}
        lo_stat = next(v for v in c if sum(u < v for u in c) <= h < sum(u <= v for u in c))
        if n % 2 == 1:
            out[k] = lo_stat
        else:
            hi_stat = next(v for v in c if sum(u < v for u in c) <= h + 1 < sum(u <= v for u in c))
            out[k] = _f32((lo_stat + hi_stat) * 0.5)
    return out


def average(x):
    x = np.asarray(x, np.float32)
    return np.array([_mean_f32(x[:, k]) for k in range(x.shape[1])], np.float32)


def trimmed_mean(x, f):
    x = np.asarray(x, np.float32)
    n, d = x.shape
    out = np.empty(d, np.float32)
    for k in range(d):
        vals = [_canon(x[i, k]) for i in range(n)]
        for _ in range(f):
            vals.remove(min(vals))
            vals.remove(max(vals))
        out[k] = _mean_f32(vals)
    return out


def trimmed_membership(x, f):
    """Rank counting instead of sorting: input i is kept at coordinate k iff
    f <= #{j : (c_j, j) < (c_i, i)} < n - f (canonical values, ties by index)."""
    x = np.asarray(x, np.float32)
    n, d = x.shape
    out = np.zeros(d, np.uint64)
    for k in range(d):
        c = [_canon(x[i, k]) for i in range(n)]
        m = 0
        for i in range(n):
            rank = sum(1 for j in range(n) if c[j] < c[i] or (c[j] == c[i] and j < i))
            if f <= rank < n - f:
                m |= 1 << i
        out[k] = m
    return out


def distances(x):
    """Exact squared Euclidean distances (Fraction), then rounded to fp64;
    non-finite or > FLT_MAX -> +inf (R4)."""
    x = np.asarray(x, np.float32)
    n, d = x.shape
    D = np.zeros((n, n), np.float64)
    flt_max = float(np.finfo(np.float32).max)
    for i in range(n):
        for j in range(i + 1, n):
            if not (np.all(np.isfinite(x[i])) and np.all(np.isfinite(x[j]))):
                v = math.inf
            else:
                s = sum((Fraction(float(a)) - Fraction(float(b))) ** 2 for a, b in zip(x[i], x[j]))
                v = float(s)
                if v > flt_max:
                    v = math.inf
            D[i, j] = D[j, i] = v
    return D


def krum_score(D, i, pool, k):
    """min over all k-subsets of pool minus {i} of the summed distances."""
    others = [j for j in pool if j != i]
    if k <= 0:
        return 0.0
    best = math.inf
    for S in itertools.combinations(others, k):
        s = math.fsum(D[i, j] for j in S) if all(math.isfinite(D[i, j]) for j in S) else math.inf
        best = min(best, s)
    return best


def multi_krum_select(D, f, m):
    n = D.shape[0]
    scores = [krum_score(D, i, range(n), n - f - 2) for i in range(n)]
    order = sorted(range(n), key=lambda i: (scores[i], i))
    return np.array(order[:m], np.int32), np.array(scores)


def bulyan_select(D, f):
    n = D.shape[0]
    pool = list(range(n))
    sel = []
    for _ in range(n - 2 * f):
        k = max(len(pool) - f - 2, 0)
        scores = {i: krum_score(D, i, pool, k) for i in pool}
        best = min(pool, key=lambda i: (scores[i], i))
        sel.append(best)
        pool.remove(best)
    return np.array(sel, np.int32)


def bulyan_coordinate_phase(x, f, sel):
    x = np.asarray(x, np.float32)
    theta = len(sel)
    beta = theta - 2 * f
    out = np.empty(x.shape[1], np.float32)
    for k in range(x.shape[1]):
        y = [_canon(x[s, k]) for s in sel]
        med = float(median(np.array(y, np.float32).reshape(-1, 1))[0])
        c = []
        for v in y:
            c.append(0.0 if v == med else _f32(abs(np.float32(v) - np.float32(med))))
        keys = [(c[t], int(sel[t])) for t in range(theta)]
        kept = [y[t] for t in range(theta) if sum(keys[u] < keys[t] for u in range(theta)) < beta]
        assert len(kept) == beta
        out[k] = _mean_f32(sorted(kept))
    return out


def mean_of_rows(x, rows):
    x = np.asarray(x, np.float32)
    return average(x[sorted(int(r) for r in rows)])


def bulyan(x, f):
    D = distances(x)
    sel = bulyan_select(D, f)
    return bulyan_coordinate_phase(x, f, sel), sel


def multi_krum(x, f, m=None):
    n = x.shape[0]
    m = n - f - 2 if m is None else m
    D = distances(x)
    sel, _ = multi_krum_select(D, f, m)
    return mean_of_rows(x, sel), sel


def mda(x, f):
    """Brute force over itertools.combinations with the Euclidean (square-root)
    diameter, exact fp64 distances from fsum; ties: first in lexicographic order."""
    import itertools
    import math
    x = np.asarray(x, np.float32)
    n, d = x.shape
    def dist(i, j):
        return math.sqrt(math.fsum((float(x[i, k]) - float(x[j, k])) ** 2 for k in range(d)))
    best, best_set = None, None
    for s in itertools.combinations(range(n), n - f):
        diam = max((dist(a, b) for a, b in itertools.combinations(s, 2)), default=0.0)
        if best is None or diam < best:
            best, best_set = diam, s
    return mean_of_rows(x, list(best_set)), np.array(best_set, np.int32)
