"""CPU oracle for the Garfield GAR hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2010_05888_b200`` never imports it, and it never
imports the product: the two share no code.

Thin numpy/ctypes marshalling around ``gar_oracle.cpp`` (plain C++17, fp64
arithmetic, definitions from PAPER.md §3.3 l.198-225 and the readings R1-R9 in
DESIGN.md).  ``oracle.brute`` holds independent pure-Python brute forces used
to pin it on tiny inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gar_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, INVALID, QUORUM, INVALID_M = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: status {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2, plain C++17 + std::thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i32p = ctypes.POINTER(ctypes.c_int32)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        I, L64 = ctypes.c_int, ctypes.c_int64
        sig = {
            "oracle_average": [f32p, I, L64, f32p, I],
            "oracle_median": [f32p, I, I, L64, f32p, I],
            "oracle_trimmed_mean": [f32p, I, I, L64, f32p, I],
            "oracle_trimmed_membership": [f32p, I, I, L64, ctypes.POINTER(ctypes.c_uint64), I],
            "oracle_sgd_update": [f32p, f32p, ctypes.c_float, L64, f32p],
            "oracle_distances": [f32p, I, L64, f64p, I],
            "oracle_krum_scores": [f64p, I, I, f64p],
            "oracle_multi_krum_select": [f64p, I, I, I, i32p],
            "oracle_bulyan_round_scores": [f64p, I, I, u8p, f64p],
            "oracle_bulyan_select": [f64p, I, I, i32p],
            "oracle_mean_of_rows": [f32p, I, L64, i32p, I, f32p, I],
            "oracle_bulyan_coordinate_phase": [f32p, I, I, L64, i32p, I, f32p, I],
            "oracle_multi_krum": [f32p, I, I, I, L64, f32p, i32p, f64p, I],
            "oracle_bulyan": [f32p, I, I, L64, f32p, i32p, f64p, I],
            "oracle_mda_select": [f64p, I, I, i32p],
            "oracle_mean_around_median": [f32p, I, I, L64, f32p, I],
            "oracle_mda": [f32p, I, I, L64, f32p, i32p, f64p, I],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = I
        L.oracle_median3_reorder.argtypes = [f32p, f32p]
        L.oracle_median3_reorder.restype = None
        _lib = L
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _f32(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return a


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _check(code, what):
    if code != OK:
        raise OracleError(code, what)


def average(x, threads=None):
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    _check(lib().oracle_average(_p(x, ctypes.c_float), n, d, _p(out, ctypes.c_float),
                                threads or default_threads()), "average")
    return out


def median(x, f=0, threads=None):
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    _check(lib().oracle_median(_p(x, ctypes.c_float), n, f, d, _p(out, ctypes.c_float),
                               threads or default_threads()), "median")
    return out


def trimmed_mean(x, f, threads=None):
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    _check(lib().oracle_trimmed_mean(_p(x, ctypes.c_float), n, f, d, _p(out, ctypes.c_float),
                                     threads or default_threads()), "trimmed_mean")
    return out


def trimmed_membership(x, f, threads=None):
    """uint64[d]: bit i of entry k set iff input i is kept by the trimmed mean at
    coordinate k (canonical order, ties by index; n <= 64)."""
    x = _f32(x)
    n, d = x.shape
    mask = np.empty(d, np.uint64)
    _check(lib().oracle_trimmed_membership(_p(x, ctypes.c_float), n, f, d, _p(mask, ctypes.c_uint64),
                                           threads or default_threads()), "trimmed_membership")
    return mask


def sgd_update(params, g, lr):
    """The server step x - lr * g with one rounding (fma)."""
    p = _f32(params).reshape(-1)
    gg = _f32(g).reshape(-1)
    out = np.empty_like(p)
    _check(lib().oracle_sgd_update(_p(p, ctypes.c_float), _p(gg, ctypes.c_float), float(lr), p.size,
                                   _p(out, ctypes.c_float)), "sgd_update")
    return out


def distances(x, threads=None):
    x = _f32(x)
    n, d = x.shape
    D = np.empty((n, n), np.float64)
    _check(lib().oracle_distances(_p(x, ctypes.c_float), n, d, _p(D, ctypes.c_double),
                                  threads or default_threads()), "distances")
    return D


def krum_scores(D, f):
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    s = np.empty(n, np.float64)
    _check(lib().oracle_krum_scores(_p(D, ctypes.c_double), n, f, _p(s, ctypes.c_double)),
           "krum_scores")
    return s


def multi_krum_select(D, f, m):
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    sel = np.empty(m, np.int32)
    _check(lib().oracle_multi_krum_select(_p(D, ctypes.c_double), n, f, m,
                                          _p(sel, ctypes.c_int32)), "multi_krum_select")
    return sel


def bulyan_round_scores(D, f, in_pool):
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    pool = np.ascontiguousarray(in_pool, np.uint8)
    s = np.empty(n, np.float64)
    _check(lib().oracle_bulyan_round_scores(_p(D, ctypes.c_double), n, f,
                                            _p(pool, ctypes.c_uint8), _p(s, ctypes.c_double)),
           "bulyan_round_scores")
    return s


def bulyan_select(D, f):
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    sel = np.empty(n - 2 * f, np.int32) if n - 2 * f > 0 else np.empty(0, np.int32)
    _check(lib().oracle_bulyan_select(_p(D, ctypes.c_double), n, f, _p(sel, ctypes.c_int32)),
           "bulyan_select")
    return sel


def mean_of_rows(x, rows, threads=None):
    x = _f32(x)
    n, d = x.shape
    rows = np.ascontiguousarray(rows, np.int32)
    out = np.empty(d, np.float32)
    _check(lib().oracle_mean_of_rows(_p(x, ctypes.c_float), n, d, _p(rows, ctypes.c_int32),
                                     len(rows), _p(out, ctypes.c_float),
                                     threads or default_threads()), "mean_of_rows")
    return out


def bulyan_coordinate_phase(x, f, sel, threads=None):
    x = _f32(x)
    n, d = x.shape
    sel = np.ascontiguousarray(sel, np.int32)
    out = np.empty(d, np.float32)
    _check(lib().oracle_bulyan_coordinate_phase(_p(x, ctypes.c_float), n, f, d,
                                                _p(sel, ctypes.c_int32), len(sel),
                                                _p(out, ctypes.c_float),
                                                threads or default_threads()),
           "bulyan_coordinate_phase")
    return out


def multi_krum(x, f, m=None, threads=None, return_D=False):
    x = _f32(x)
    n, d = x.shape
    m = n - f - 2 if m is None else m
    out = np.empty(d, np.float32)
    sel = np.empty(max(m, 1), np.int32)
    D = np.empty((n, n), np.float64)
    _check(lib().oracle_multi_krum(_p(x, ctypes.c_float), n, f, m, d, _p(out, ctypes.c_float),
                                   _p(sel, ctypes.c_int32), _p(D, ctypes.c_double),
                                   threads or default_threads()), "multi_krum")
    return (out, sel, D) if return_D else (out, sel)


def mean_around_median(x, f, threads=None):
    """Per coordinate, the mean of the n - 2f values closest to the median
    (Bulyan's coordinate phase over all n inputs; PAPER.md l.316 footnote)."""
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    _check(lib().oracle_mean_around_median(_p(x, ctypes.c_float), n, f, d, _p(out, ctypes.c_float),
                                           threads or default_threads()), "mean_around_median")
    return out


def sanitize(x, f):
    """(kept, excluded) input indices; a row is excluded iff it
    holds a non-finite value; more than f excluded -> OracleError(2)."""
    x = _f32(x)
    bad = [i for i in range(x.shape[0]) if not np.all(np.isfinite(x[i]))]
    if len(bad) > f:
        raise OracleError(2, "sanitize (TooManyNonFinite)")
    return [i for i in range(x.shape[0]) if i not in bad], bad


def mda_select(D, f):
    """Indices (ascending) of the size n-f subset of minimum diameter
    (max pairwise squared distance), ties to the lexicographically smallest set."""
    D = np.ascontiguousarray(D, np.float64)
    n = D.shape[0]
    sel = np.empty(max(n - f, 1), np.int32)
    _check(lib().oracle_mda_select(_p(D, ctypes.c_double), n, f, _p(sel, ctypes.c_int32)), "mda_select")
    return sel[: n - f]


def mda(x, f, threads=None, return_D=False):
    """MDA: the average of the minimum-diameter subset of n-f inputs."""
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    sel = np.empty(max(n - f, 1), np.int32)
    D = np.empty((n, n), np.float64)
    _check(lib().oracle_mda(_p(x, ctypes.c_float), n, f, d, _p(out, ctypes.c_float), _p(sel, ctypes.c_int32),
                            _p(D, ctypes.c_double), threads or default_threads()), "mda")
    return (out, sel[: n - f], D) if return_D else (out, sel[: n - f])


def krum(x, f, threads=None, return_D=False):
    return multi_krum(x, f, 1, threads, return_D)


def bulyan(x, f, threads=None, return_D=False):
    x = _f32(x)
    n, d = x.shape
    out = np.empty(d, np.float32)
    sel = np.empty(max(n - 2 * f, 1), np.int32)
    D = np.empty((n, n), np.float64)
    _check(lib().oracle_bulyan(_p(x, ctypes.c_float), n, f, d, _p(out, ctypes.c_float),
                               _p(sel, ctypes.c_int32), _p(D, ctypes.c_double),
                               threads or default_threads()), "bulyan")
    return (out, sel, D) if return_D else (out, sel)


def median3_reorder(v):
    v = np.ascontiguousarray(v, np.float32)
    w = np.empty(3, np.float32)
    lib().oracle_median3_reorder(_p(v, ctypes.c_float), _p(w, ctypes.c_float))
    return w


def widen_bf16(bits):
    """bf16 -> fp32, exactly (R16; SURVEY §8f-4 "bf16 gradient inputs").

    A bf16 value is, by definition, the upper 16 bits of an IEEE-754 binary32
    (same sign bit, same 8-bit exponent, the 7 leading fraction bits), so its
    fp32 value is the 32-bit word ``bits << 16``.  Every bf16 value (NaN, +-inf,
    +-0 and subnormals included) is representable in fp32; the widening rounds
    nothing.  Reading R16: a rule over bf16 inputs is the fp32 rule over the
    widened values, so the oracle of a bf16 call is this widening followed by
    the fp32 oracle below -- no other arithmetic changes."""
    b = np.ascontiguousarray(bits)
    if b.dtype != np.uint16:
        raise TypeError("bf16 inputs are given as their uint16 bit patterns")
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def aggregate_bf16(rule, bits, f, m=None, threads=None):
    """aggregate() of bf16 inputs (uint16 bit patterns [n, d]): R16."""
    return aggregate(rule, widen_bf16(bits), f, m, threads)


def aggregate(rule, x, f, m=None, threads=None):
    """Dispatch by rule name (test convenience). Returns (out, selected or None)."""
    if rule == "average":
        return average(x, threads), None
    if rule == "median":
        return median(x, f, threads), None
    if rule == "trimmed_mean":
        return trimmed_mean(x, f, threads), None
    if rule == "krum":
        return krum(x, f, threads)
    if rule == "multi_krum":
        return multi_krum(x, f, m, threads)
    if rule == "bulyan":
        return bulyan(x, f, threads)
    raise ValueError(rule)
