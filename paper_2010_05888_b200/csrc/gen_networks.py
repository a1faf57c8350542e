#!/usr/bin/env python3
"""Generate ``networks.cuh``: straight-line compare-exchange networks for the
coordinate-selection kernel (product code; shares nothing with oracle/).

For every size N in 1..64 we take four constructions: Batcher's odd-even
merge sort, the bitonic sort and Parberry's pairwise network on the next power
of two P >= N (wires N..P-1 hold the constant +inf, and the padding is
constant-propagated: a comparator against a +inf wire is a no-op or a
relabel), and Batcher's merge exchange on exactly N wires.  Only the min/max
outputs that reach the requested output positions are kept, and the cheapest
construction (in emitted min/max instructions) wins per (N, outputs).

Emitted functions (all in-place on ``T v[N]``, ascending order; T = float, or
``bf2`` = two bf16 values of adjacent coordinates in one 32-bit register, whose
compare-exchange is one packed min.bf16x2 / max.NaN.bf16x2 pair — elem.cuh):

* ``gar_net::sort_<N>(v)``    — full sort, every position valid;
* ``gar_net::median_<N>(v)``  — only v[(N-1)/2] (and v[N/2] for even N) valid;
* ``gar_net::trim_<N>(v)``    — v[F..N-F-1] valid and sorted, F = trim_f<N>() =
  max(0, (N-3)/4): the trimmed mean at the paper's f for n = 4f+3;
* ``gar_net::window_<N>(v)``  — odd N >= 5: v[h-2..h+2] valid and sorted,
  h = (N-1)/2: Bulyan's coordinate phase when beta = 3 (n = 4f+3).

Compare-exchange = vmin (fminf / min.bf16x2: drops a NaN operand) + vmax_nan
(max.NaN: returns NaN if either operand is NaN).  With these two, a NaN moves through
the network exactly like +inf (R1: NaN orders as +inf): min(NaN, x) = x,
max(NaN, x) = NaN, min/max(NaN, NaN) = NaN.  So inputs need no
canonicalisation; the kernel maps NaN -> +inf only on the outputs it uses.
-0 and +0 compare equal (they may swap, which no result can observe).
"""
from __future__ import annotations

import os
import sys

MAXN = 64


def oddeven_merge_sort(P):
    """Batcher's odd-even merge sort comparators for P = 2^k wires."""
    comps = []

    def merge(lo, n, r):
        step = r * 2
        if step < n:
            merge(lo, n, step)
            merge(lo + r, n, step)
            for i in range(lo + r, lo + n - r, step):
                comps.append((i, i + r))
        else:
            comps.append((lo, lo + r))

    def sort(lo, n):
        if n > 1:
            m = n // 2
            sort(lo, m)
            sort(lo + m, m)
            merge(lo, n, 1)

    sort(0, P)
    return comps


def bitonic_sort(P):
    comps = []
    k = 2
    while k <= P:
        j = k // 2
        while j > 0:
            for i in range(P):
                l = i ^ j
                if l > i:
                    if (i & k) == 0:
                        comps.append((i, l))
                    else:
                        comps.append((l, i))   # descending block: min goes to l
            j //= 2
        k *= 2
    return comps


def merge_exchange(N):
    """Batcher's merge exchange for any N (Knuth, TAOCP 5.2.2, Algorithm M):
    no padding wires."""
    comps = []
    t = 1
    while (1 << t) < N:
        t += 1
    p = 1 << (t - 1)
    while p > 0:
        q, r, dd = 1 << (t - 1), 0, p
        while True:
            for i in range(N - dd):
                if (i & p) == r:
                    comps.append((i, i + dd))
            if q == p:
                break
            dd, q, r = q - p, q >> 1, p
        p >>= 1
    return comps


def pairwise_sort(P):
    """Parberry's pairwise sorting network for P = 2^k wires."""
    comps = []
    a = 1
    while a < P:
        b, c = a, 0
        while b < P:
            comps.append((b - a, b))
            b += 1
            c = (c + 1) % a
            if c == 0:
                b += a
        a *= 2
    a //= 4
    e = 1
    while a > 0:
        d = e
        while d > 0:
            b, c = (d + 1) * a, 0
            while b < P:
                comps.append((b - d * a, b))
                b += 1
                c = (c + 1) % a
                if c == 0:
                    b += a
            d //= 2
        a //= 2
        e = e * 2 + 1
    return comps


def build_ssa(N, comps):
    """Symbolic execution.  Wire contents are ('in', i), ('inf',) or ('op', id).
    Returns (ops, final) where ops[id] = (kind, a, b) with kind in {min,max}."""
    P = 1
    while P < N:
        P *= 2
    wires = [("in", i) if i < N else ("inf",) for i in range(P)]
    ops = []
    for (i, j) in comps:
        a, b = wires[i], wires[j]
        if a == ("inf",) and b == ("inf",):
            continue
        if b == ("inf",):
            continue                      # min(a, inf) = a stays at i, inf at j
        if a == ("inf",):
            wires[i], wires[j] = b, a     # relabel
            continue
        ops.append(("min", a, b))
        mn = ("op", len(ops) - 1)
        ops.append(("max", a, b))
        mx = ("op", len(ops) - 1)
        wires[i], wires[j] = mn, mx
    return ops, wires[:N]


def live_ops(ops, outputs):
    live = set()
    stack = [o for o in outputs if o[0] == "op"]
    while stack:
        o = stack.pop()
        if o[1] in live:
            continue
        live.add(o[1])
        _, a, b = ops[o[1]]
        for x in (a, b):
            if x[0] == "op":
                stack.append(x)
    return live


def best_network(N, positions):
    P = 1
    while P < N:
        P *= 2
    best = None
    for name, comps in (("oddeven", oddeven_merge_sort(P)), ("bitonic", bitonic_sort(P)),
                        ("merge-exchange", merge_exchange(N)), ("pairwise", pairwise_sort(P))):
        ops, final = build_ssa(N, comps)
        live = live_ops(ops, [final[p] for p in positions])
        cost = len(live)
        if best is None or cost < best[0]:
            best = (cost, name, ops, final, live)
    return best


def verify(N, ops, final, positions, trials=2000):
    import random
    rnd = random.Random(N)
    for t in range(trials):
        if N <= 12 and t < (1 << N):
            vals = [(t >> i) & 1 for i in range(N)]          # 0-1 principle, exhaustive
        else:
            vals = [rnd.randint(-5, 5) for _ in range(N)]
        res = {}

        def ev(x):
            if x[0] == "in":
                return vals[x[1]]
            if x[0] == "inf":
                return float("inf")
            if x[1] not in res:
                k, a, b = ops[x[1]]
                res[x[1]] = min(ev(a), ev(b)) if k == "min" else max(ev(a), ev(b))
            return res[x[1]]

        ref = sorted(vals)
        for p in positions:
            assert ev(final[p]) == ref[p], (N, p)


def emit(N, fname, positions):
    cost, name, ops, final, live = best_network(N, positions)
    verify(N, ops, final, positions, trials=600 if N > 12 else (1 << N))
    what = "full sort" if len(positions) == N else ("median" if len(positions) <= 2 else
                                                       f"positions {positions[0]}..{positions[-1]}")
    if len(positions) == N and N <= 2:
        what = "full sort"
    lines = [f"// N={N}: {name}, {cost} min/max ({what})",
             f"template <class T> __device__ __forceinline__ void {fname}_{N}(T* v) {{"]
    names = {}

    def ref(x):
        if x[0] == "in":
            return f"v{x[1]}"
        return names[x[1]]

    for i in range(N):
        lines.append(f"  const T v{i} = v[{i}];")
    for k, (kind, a, b) in enumerate(ops):
        if k not in live:
            continue
        nm = f"t{k}"
        names[k] = nm
        fn = "vmin" if kind == "min" else "vmax_nan"
        lines.append(f"  const T {nm} = {fn}({ref(a)}, {ref(b)});")
    for p in positions:
        lines.append(f"  v[{p}] = {ref(final[p])};")
    lines.append("}")
    return "\n".join(lines), cost


def trim_f(N):
    return (N - 3) // 4 if N >= 3 else 0


def main(out_path):
    parts = ["// GENERATED by gen_networks.py — do not edit.  Product code (libgar);",
             "// shares nothing with oracle/.  Pruned Batcher / bitonic / pairwise /",
             "// merge-exchange networks with +inf padding constant-propagated",
             "// (DESIGN.md §4.1, coord_select).",
             "#pragma once", "#include \"elem.cuh\"", "namespace gar_net {",
             "using gar::vmin;", "using gar::vmax_nan;"]
    table = []
    for N in range(1, MAXN + 1):
        src, c_sort = emit(N, "sort", list(range(N)))
        parts.append(src)
        med = [(N - 1) // 2] if N % 2 else [N // 2 - 1, N // 2]
        src, c_med = emit(N, "median", med)
        parts.append(src)
        F = trim_f(N)
        src, c_trim = emit(N, "trim", list(range(F, N - F)))
        parts.append(src)
        if N % 2 == 1 and N >= 5:
            h = (N - 1) // 2
            src, _ = emit(N, "window", list(range(h - 2, h + 3)))
            parts.append(src)
        table.append((N, c_sort, c_med, c_trim))
    parts.append("template <int N> constexpr int trim_f() { return N >= 3 ? (N - 3) / 4 : 0; }")
    parts.append("template <int N> struct Net;")
    for N in range(1, MAXN + 1):
        body = (f"template <> struct Net<{N}> {{ "
                f"template <class T> static __device__ __forceinline__ void sort(T* v) {{ sort_{N}(v); }} "
                f"template <class T> static __device__ __forceinline__ void median(T* v) {{ median_{N}(v); }} "
                f"template <class T> static __device__ __forceinline__ void trim(T* v) {{ trim_{N}(v); }}")
        if N % 2 == 1 and N >= 5:
            body += f" template <class T> static __device__ __forceinline__ void window(T* v) {{ window_{N}(v); }}"
        parts.append(body + " };")
    for k in ("sort", "median", "trim", "window"):
        parts.append(f"template <int N, class T> __device__ __forceinline__ void {k}_net(T* v) {{ Net<N>::{k}(v); }}")
    parts.append("// min/max instruction counts (N, sort, median, trim at F = trim_f<N>):")
    for N, a, b, c in table:
        parts.append(f"//   {N:2d} {a:4d} {b:4d} {c:4d}")
    parts.append("}  // namespace gar_net")
    with open(out_path, "w") as fh:
        fh.write("\n".join(parts) + "\n")


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.abspath(__file__)), "networks.cuh")
    main(out)
