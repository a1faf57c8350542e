"""The paper's two-call interface, ``init(name, n, f)`` / ``aggregate(tensors)``
(§4.1 "Aggregation"), over libgar.

The Aggregator caches its device workspace (the paper's "allocating space only
for one iteration along with the intermediate selected gradients", l.401:
here one n x n Gram per CTA plus the selected indices).
"""
from __future__ import annotations

import torch

from . import _lib


class Aggregator:
    def __init__(self, rule: str, n: int, f: int, m: int | None = None):
        self.rule = rule
        self.rid = _lib.rule_id(rule)
        self.n, self.f = int(n), int(f)
        self.m = 0 if m is None else int(m)
        # the library's own argument check (quorum, m, MDA budget) without touching the GPU
        code = _lib.gar_check_args(rule, self.n, self.f, self.m)
        if code != 0:
            raise _lib.GarError(code, f"init({rule!r}, n={n}, f={f}, m={m})")
        self._ws = {}
        self._idx = {}

    @property
    def num_selected(self) -> int:
        return _lib.gar_num_selected(self.rule, self.n, self.f, self.m)

    def workspace(self, device) -> torch.Tensor | None:
        nbytes = _lib.gar_workspace_bytes(self.rule, self.n, self.f, 0)
        if nbytes == 0:
            return None
        key = str(device)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._ws[key] = ws
        return ws

    def indices_buffer(self, device) -> torch.Tensor:
        key = str(device)
        t = self._idx.get(key)
        if t is None:
            t = torch.empty(_lib.MAX_N, dtype=torch.int32, device=device)
            self._idx[key] = t
        return t

    def _check_n(self, grads):
        n = grads.shape[0] if isinstance(grads, torch.Tensor) else len(grads)   # tensors, lists, DevicePtrRows
        if n != self.n:
            raise ValueError(f"expected n = {self.n} gradients, got {n}")

    def aggregate(self, grads, out: torch.Tensor | None = None, d: int | None = None,
                  indices: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """out (fp32[d]) = GAR(grads); grads: list of n CUDA fp32 (or bf16) vectors or an
        [n, ld] matrix.  bf16 inputs are widened exactly to fp32 (R16)."""
        self._check_n(grads)
        arr, n, d, dev, dt = _lib.row_pointers_dt(grads, d)
        if out is None:
            out = torch.empty(d, dtype=torch.float32, device=dev)
        ws = self.workspace(dev)
        wsb = 0 if ws is None else ws.numel()
        o = _lib._buf(out, torch.float32, d, dev, "out")
        ix = _lib._idx(indices, self.rule, n, self.f, self.m, dev, True)
        if dt == 0:
            _lib.check(_lib.lib.gar_aggregate_ex(self.rid, arr, n, self.f, self.m, d, o, ix, _lib._ptr(ws), wsb,
                                                 _lib.stream_handle(dev, stream)), f"aggregate[{self.rule}]")
        else:
            _lib.check(_lib.lib.gar_aggregate_dt(self.rid, dt, arr, n, self.f, self.m, d, o, ix, _lib._ptr(ws), wsb,
                                                 _lib.stream_handle(dev, stream)), f"aggregate[{self.rule}]")
        return out

    def graphed(self, grads, out: torch.Tensor, d: int | None = None, indices: torch.Tensor | None = None):
        """A CUDA graph of aggregate(grads, out) for fixed buffers: the
        returned callable replays the whole kernel sequence (Gram, reduction,
        selection, combine, or the coordinate kernel) with one launch, which
        is what small, launch-bound configurations (d ~ 1e5) need.  The
        gradient buffers and `out` must stay allocated and at the same
        addresses; their contents may change between replays."""
        self._check_n(grads)
        dev = grads.device if isinstance(grads, torch.Tensor) else grads[0].device
        self.aggregate(grads, out=out, d=d, indices=indices)          # warm-up: workspace, attributes, caches
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                self.aggregate(grads, out=out, d=d, indices=indices)
        torch.cuda.current_stream(dev).wait_stream(side)
        return graph.replay

    def select(self, grads, d: int | None = None, stream=None) -> torch.Tensor:
        """Selected input indices (device int32), in selection order."""
        self._check_n(grads)
        arr, n, d, dev, dt = _lib.row_pointers_dt(grads, d)
        ws = self.workspace(dev)
        if ws is None:
            raise _lib.GarError(5, f"select[{self.rule}]")
        idx = torch.empty(_lib.MAX_N, dtype=torch.int32, device=dev)
        sel = _lib.gar_select if dt == 0 else _lib.gar_select_dt
        nsel = sel(self.rule, grads, self.f, self.m, idx, ws, d=d, stream=stream)
        return idx[:nsel]


    def aggregate_sharded(self, rows_local, d: int, group=None, output: str = "replicated"):
        """Multi-GPU form (one process per GPU, d sharded): rows_local is this
        rank's slice [n, >= d_local] of every gradient (dist.shard_bounds gives
        the slice); returns the aggregate of the whole d-dimensional vectors,
        replicated on every rank (or this rank's slice with output="sharded").
        See dist.ShardedAggregator."""
        from .dist import ShardedAggregator
        key = (int(d), id(group), output)
        sh = getattr(self, "_sharded", {})
        if key not in sh:
            sh[key] = ShardedAggregator(self.rule, self.n, self.f, d, m=self.m or None, group=group, output=output)
            self._sharded = sh
        return sh[key].aggregate(rows_local)


class TooManyNonFinite(ValueError):
    """more than f inputs hold non-finite values."""


def sanitize(grads, f: int, d: int | None = None, stream=None):
    """SPEC S:43-51 (vector-level sanitize): (kept, excluded)
    input indices, excluded = the rows holding any NaN / +-inf, found by
    gar_nonfinite_rows on the GPU (one pass over the inputs, then one 8-byte
    read back to the host).  Raises TooManyNonFinite if more than f."""
    arr, n, d, dev = _lib.row_pointers(grads, d)
    mask = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.gar_nonfinite_rows(grads, mask, d=d, stream=stream)
    m = int(mask.item()) & ((1 << 64) - 1)
    excluded = [i for i in range(n) if (m >> i) & 1]
    if len(excluded) > f:
        raise TooManyNonFinite(f"{len(excluded)} inputs hold non-finite values, more than f = {f}")
    return [i for i in range(n) if not (m >> i) & 1], excluded


def _select_rows(grads, idx):
    if isinstance(grads, torch.Tensor):
        base, rs = grads.data_ptr(), grads.stride(0) * 4
        return _lib.DevicePtrRows([base + i * rs for i in idx], grads.device)
    if isinstance(grads, _lib.DevicePtrRows):
        return _lib.DevicePtrRows([grads.ptrs[i] for i in idx], grads.device)
    return [grads[i] for i in idx]


def aggregate_sanitized(agg: "Aggregator", grads, out: torch.Tensor | None = None, d: int | None = None,
                        indices: torch.Tensor | None = None):
    """SPEC's AggregationOutcome path: drop the non-finite inputs (they count
    toward f: the rule runs on n - e inputs with f - e), aggregate the rest.
    Returns (out, excluded indices).  indices (optional, Krum family / MDA):
    receives the selection, numbered among the kept inputs."""
    kept, excluded = sanitize(grads, agg.f, d)
    if not excluded:
        return agg.aggregate(grads, out=out, d=d, indices=indices), excluded
    e = len(excluded)
    sub = Aggregator(agg.rule, agg.n - e, agg.f - e, (agg.m or None) if agg.rule == "multi_krum" else None)
    dd = d if d is not None else _lib.row_pointers(grads)[2]
    return sub.aggregate(_select_rows(grads, kept), out=out, d=dd, indices=indices), excluded


def init(name: str, n: int, f: int, m: int | None = None) -> Aggregator:
    """"The init() function takes the name of the required GAR
    (e.g., "median"), the value of n, the total number of inputs, and f"."""
    return Aggregator(name, n, f, m)
