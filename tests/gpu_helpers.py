"""Shared helpers for the GPU parity tests (CUDA path vs oracle)."""
from __future__ import annotations

import numpy as np
import torch

import oracle

KRUM_FAMILY = ("krum", "multi_krum", "bulyan")
EPS_TIE = 1e-5          # selection-parity rule: relative score slack


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


def distances_close(D_gpu: np.ndarray, D_ref: np.ndarray, rtol: float = 1e-5):
    fin = np.isfinite(D_ref)
    assert np.array_equal(np.isfinite(D_gpu), fin), "non-finite pattern differs"
    pos = D_ref[fin & (D_ref > 0)]
    floor = 1e-9 * (np.median(pos) if pos.size else 0.0)
    err = np.abs(D_gpu[fin] - D_ref[fin])
    tol = rtol * D_ref[fin] + floor
    assert np.all(err <= tol), f"max rel err {np.max(err / np.maximum(D_ref[fin], 1e-300)):.3e}"
    return float(np.max(err / np.maximum(D_ref[fin], floor if floor > 0 else 1e-300)))
