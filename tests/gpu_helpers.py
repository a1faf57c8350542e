"""Shared helpers for the GPU parity tests (CUDA path vs oracle)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

KRUM_FAMILY = ("krum", "multi_krum", "bulyan")
EPS_TIE = 1e-5          # selection-parity rule: relative score slack
SEPARATED = 1e-4        # oracle score gaps above this make a decision well posed
# selection verdicts of this session ({verdict: count}); printed by conftest at the end
VERDICTS: dict = {}


def to_device(x: np.ndarray) -> torch.Tensor:
    """[n, d] fp32 host matrix -> [n, ld] CUDA matrix with 16-byte aligned rows."""
    n, d = x.shape
    ld = (d + 3) // 4 * 4
    X = torch.zeros((n, ld), dtype=torch.float32)
    X[:, :d] = torch.from_numpy(np.ascontiguousarray(x, np.float32))
    return X.cuda()


def assert_same_bits(got: np.ndarray, ref: np.ndarray, what: str = ""):
    """Bit-exact equality, treating any two NaNs as equal."""
    got = np.asarray(got, np.float32)
    ref = np.asarray(ref, np.float32)
    assert got.shape == ref.shape
    gn, rn = np.isnan(got), np.isnan(ref)
    bad = (gn != rn) | (~gn & (got.view(np.uint32) != ref.view(np.uint32)))
    if bad.any():
        k = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} differ, e.g. at {k.tolist()}: "
                             f"gpu {got[k].tolist()} vs oracle {ref[k].tolist()}")


def check_selection(rule, D_oracle: np.ndarray, f: int, m: int, sel_gpu: np.ndarray) -> str:
    """'exact' if the GPU selection equals the oracle's; 'eps-tie' if every GPU
    choice is within EPS_TIE of the oracle's best score at that step (rounds
    replayed with the GPU's previous choices forced); raises otherwise."""
    n = D_oracle.shape[0]
    sel_gpu = [int(v) for v in sel_gpu]
    if rule == "bulyan":
        ref = oracle.bulyan_select(D_oracle, f).tolist()
        if sel_gpu == ref:
            return "exact"
        pool = np.ones(n, np.uint8)
        for t, pick in enumerate(sel_gpu):
            s = oracle.bulyan_round_scores(D_oracle, f, pool)
            assert pool[pick], f"round {t}: GPU picked {pick} twice"
            best = np.nanmin(s)
            assert s[pick] <= best * (1 + EPS_TIE) + 1e-300, \
                f"bulyan round {t}: gpu pick {pick} score {s[pick]!r} vs best {best!r} (oracle {ref})"
            pool[pick] = 0
        return "eps-tie"
    ref = oracle.multi_krum_select(D_oracle, f, m).tolist()
    if sel_gpu == ref:
        return "exact"
    s = oracle.krum_scores(D_oracle, f)
    order = sorted(range(n), key=lambda i: (s[i], i))
    assert len(set(sel_gpu)) == len(sel_gpu)
    for t, pick in enumerate(sel_gpu):
        # the t-th GPU pick must tie (within EPS) with the t-th oracle score
        assert abs(s[pick] - s[order[t]]) <= EPS_TIE * abs(s[order[t]]) + 1e-300, \
            f"{rule} position {t}: gpu {pick} ({s[pick]!r}) vs oracle {order[t]} ({s[order[t]]!r})"
    return "eps-tie"


def decision_gap(rule, D_oracle: np.ndarray, f: int, m: int) -> float:
    """The smallest relative score gap over the oracle's selection decisions:
    Multi-Krum: between consecutive sorted scores at positions 0..m (the m
    picks and the first rejected); Bulyan: per round, between the best and
    second-best score of the pool.  Exact ties (bitwise-equal oracle scores:
    rounds with zero neighbours, where every score is 0, or structurally equal
    sums such as the shared nearest pair D_ij = D_ji with one neighbour) are
    decided by the lower-index rule, not by a score difference, and are
    skipped: the GPU must reproduce them too.  Above SEPARATED, anything but an
    exact GPU selection is a bug."""
    n = D_oracle.shape[0]
    gap = np.inf
    if rule == "bulyan":
        pool = np.ones(n, np.uint8)
        for _ in range(n - 2 * f):
            members = np.flatnonzero(pool)
            s = oracle.bulyan_round_scores(D_oracle, f, pool)
            ss = sorted((s[i], i) for i in members)
            if len(members) - f - 2 > 0 and len(ss) > 1 and ss[1][0] != ss[0][0]:
                gap = min(gap, (ss[1][0] - ss[0][0]) / max(abs(ss[1][0]), 1e-300))
            pool[ss[0][1]] = 0
        return gap
    s = oracle.krum_scores(D_oracle, f)
    if n - f - 2 <= 0:
        return gap
    o = sorted(range(n), key=lambda i: (s[i], i))
    for t in range(min(m, n - 1)):
        if s[o[t + 1]] != s[o[t]]:
            gap = min(gap, (s[o[t + 1]] - s[o[t]]) / max(abs(s[o[t + 1]]), 1e-300))
    return gap


def assert_selection(rule, D_oracle: np.ndarray, f: int, m: int, sel_gpu: np.ndarray,
                     require_separated: bool = False) -> str:
    """The strict selection check: the GPU selection must
    be exactly the oracle's whenever the oracle's decisions are separated by
    more than SEPARATED; an eps-tie verdict is accepted only for inputs whose
    decision gap is below that (and tallied).  require_separated: the input
    claims to be well separated (synth kind="separated"); assert that too."""
    gap = decision_gap(rule, D_oracle, f, m)
    if require_separated:
        assert gap > SEPARATED, f"{rule}: input not well separated (gap {gap:.3e})"
    verdict = check_selection(rule, D_oracle, f, m, sel_gpu)
    if gap > SEPARATED:
        assert verdict == "exact", f"{rule}: well-separated selection (gap {gap:.3e}) not exact: {list(sel_gpu)}"
    VERDICTS[verdict] = VERDICTS.get(verdict, 0) + 1
    return verdict


def distances_close(D_gpu: np.ndarray, D_ref: np.ndarray, rtol: float = 1e-5):
    fin = np.isfinite(D_ref)
    assert np.array_equal(np.isfinite(D_gpu), fin), "non-finite pattern differs"
    pos = D_ref[fin & (D_ref > 0)]
    floor = 1e-9 * (np.median(pos) if pos.size else 0.0)
    err = np.abs(D_gpu[fin] - D_ref[fin])
    tol = rtol * D_ref[fin] + floor
    assert np.all(err <= tol), f"max rel err {np.max(err / np.maximum(D_ref[fin], 1e-300)):.3e}"
    return float(np.max(err / np.maximum(D_ref[fin], floor if floor > 0 else 1e-300)))
