"""d-sharded multi-GPU aggregation (north_star "Partitioning
across the 8xB200 box by sharding d").

Rank r of G holds coordinates [lo_r, hi_r) of every one of the n gradients
(``shard_bounds``: contiguous slices, boundaries at multiples of 1024
coordinates).  Then:

* Average / Median / trimmed mean and the Bulyan coordinate phase are purely
  per-coordinate: each rank aggregates its own slice, no communication;
* Krum / Multi-Krum / Bulyan need the n x n distance matrix of the WHOLE
  vectors: each rank computes the partial Gram matrix of its slice and the
  ranks sum them (the centring of the Gram is per coordinate, so partial
  Grams of disjoint slices add up exactly).  By default the sum is fused into
  the Gram's own kernels over NVLink peer memory (``gar_gram_exchange``: the
  reduced partial is stored into every rank's symmetric slot array, a flag
  handshake, a rank-ordered sum -- no collective library call); or
  ``gar_gram_partial`` + one NCCL all-reduce (``exchange="nccl"``).  Every
  rank then runs the identical deterministic selection
  (``gar_select_from_gram``) and combines its own slice (``gar_combine``);
* the aggregate is all-gathered (``output="replicated"``: NCCL all-gather
  after the kernel, the north_star default), written by the producing kernel
  itself into every GPU's output buffer over NVLink (``output="fused"``:
  torch symmetric memory, one store per peer, ``gar_*_bcast``; or with
  ``"fused-mc"`` one NVLink SHARP multicast store per result, ``gar_*_mcast``;
  then one device-side barrier), all-gathered by NCCL asynchronously so the
  transfer overlaps the caller's next work (``"replicated-async"``, then
  ``wait()``), or left d-sharded (``output="sharded"``, what a ZeRO-style
  optimizer consumes).

The paper's own exchange is PyTorch ``broadcast``/``gather`` over NCCL or gloo
(§4.2); here the only collectives are one tiny
all-reduce per Krum-family call and the optional output all-gather.

The kernels are reached through ``backend`` (default: libgar).  Tests inject a
host-side stand-in to exercise the sharding and exchange logic over gloo on CPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

KRUM_FAMILY = ("krum", "multi_krum", "bulyan", "mda")     # the Gram-based selection rules


def shard_bounds(d: int, rank: int, world: int, align: int = 1024) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of rank `rank`; every slice but the last has
    the same length, a multiple of `align` coordinates (16-byte row alignment)."""
    per = (d + world - 1) // world
    per = (per + align - 1) // align * align
    lo = min(d, rank * per)
    hi = min(d, lo + per)
    return lo, hi


def shard_len(d: int, world: int, align: int = 1024) -> int:
    return shard_bounds(d, 0, world, align)[1] if world > 1 else d


def is_bf16(rows) -> bool:
    """bf16 gradient rows: a bf16 tensor or a list of them."""
    t = rows if isinstance(rows, torch.Tensor) else (rows[0] if isinstance(rows, (list, tuple)) and rows else None)
    return t is not None and t.dtype == torch.bfloat16


class _LibgarBackend:
    """The product kernels (libgar C ABI).  bf16 rows go through the _dt entry
    points (exact widening, R16); the peer-memory exchange and the
    fused outputs are fp32-only, so bf16 rows use the NCCL exchange and a
    separate all-gather."""

    def __init__(self):
        from . import _lib
        self._lib = _lib

    def coordinatewise(self, agg, rows, out, d):
        agg.aggregate(rows, out=out, d=d)

    def gram_partial(self, rows, gram, ws, d):
        if is_bf16(rows):
            self._lib.gar_gram_partial_dt(rows, gram, ws, d=d)
        else:
            self._lib.gar_gram_partial(rows, gram, ws, d=d)

    def select_from_gram(self, rule, gram, n, f, m, idx, ws=None):
        return self._lib.gar_select_from_gram(rule, gram, n, f, m, idx, workspace=ws)

    def gram_exchange(self, rows, gram, ws, d, slots, flags, rank, world, epoch, stage=None):
        self._lib.gar_gram_exchange(rows, gram, ws, slots, flags, rank, world, epoch, d=d, stage=stage)

    def combine(self, rule, rows, f, m, idx, out, d, extra=()):
        if is_bf16(rows):
            if extra:
                raise NotImplementedError("fused outputs take fp32 rows; use output='replicated' for bf16")
            self._lib.gar_combine_dt(rule, rows, f, m, idx, out, d=d)
        elif isinstance(extra, Multicast):
            self._lib.gar_combine_mcast(rule, rows, f, m, idx, out, extra.addr, d=d)
        elif extra:
            self._lib.gar_combine_bcast(rule, rows, f, m, idx, out, extra, d=d)
        else:
            self._lib.gar_combine(rule, rows, f, m, idx, out, d=d)

    def coordinatewise_bcast(self, agg, rows, out, d, extra):
        if isinstance(extra, Multicast):
            self._lib.gar_aggregate_mcast(agg.rule, rows, agg.f, agg.m, out, extra.addr, workspace=None, d=d)
        else:
            self._lib.gar_aggregate_bcast(agg.rule, rows, agg.f, agg.m, out, extra, workspace=None, d=d)


class Multicast:
    """Fused-output destination given as one multicast (NVLS) address: the
    kernel's multimem stores reach every rank's buffer, this rank's included."""

    def __init__(self, addr: int):
        self.addr = int(addr)

    def __bool__(self):
        return True


class ShardedAggregator:
    """``init(name, n, f)`` / ``aggregate`` over a d-sharded
    process group: one process per GPU, each holding its slice of every row."""

    def __init__(self, rule: str, n: int, f: int, d: int, m: int | None = None, group=None,
                 output: str = "replicated", backend=None, exchange: str = "auto"):
        if output not in ("replicated", "replicated-async", "sharded", "fused", "fused-mc"):
            raise ValueError(output)
        self.rule, self.n, self.f, self.d = rule, int(n), int(f), int(d)
        self.m = 0 if m is None else int(m)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.lo, self.hi = shard_bounds(self.d, self.rank, self.world) if self.world > 1 else (0, self.d)
        self.d_local = self.hi - self.lo
        self.per = shard_len(self.d, self.world)
        self.output = output
        self.backend = backend if backend is not None else _LibgarBackend()
        # Krum-family Gram exchange: "peer" = gar_gram_exchange over symmetric
        # memory (one fused reduce + peer stores + flag handshake, no NCCL),
        # "nccl" = gar_gram_partial + NCCL all-reduce; "auto" = peer when the
        # backend has it and the group is on CUDA devices.
        if exchange not in ("auto", "peer", "nccl"):
            raise ValueError(exchange)
        self.exchange = exchange
        self._xchg = None          # (symmetric buffer, handle, epoch) for the peer exchange
        self._agg = None
        self._ws = None
        self._gram = None
        self._idx = None
        self._pad = None
        self._symm = None          # (symmetric out_full, handle, Multicast | peer addresses) for fused output

    def _fused_buffers(self, device):
        """Replicated output in symmetric memory, and where the kernel stores
        this rank's slice: the slice's addresses in every OTHER rank's buffer
        (peer-mapped over NVLink, one store per peer), or with
        output="fused-mc" and a multicast-capable group the multicast address
        of the slice (NVLS: one store per result, replicated by the NVSwitch;
        measured slower than the peer stores on B200, profiles/)."""
        if self._symm is None:
            import torch.distributed._symmetric_memory as symm_mem
            # two output buffers, alternating per call, so a deferred barrier
            # (aggregate(barrier=False) + sync()) cannot let a rank that runs
            # one call ahead overwrite an output another rank may still read
            bufs = []
            group = self.group if self.group is not None else dist.group.WORLD
            for _ in range(2):
                buf = symm_mem.empty(self.per * self.world, dtype=torch.float32, device=device)
                handle = symm_mem.rendezvous(buf, group)
                mc = int(handle.multicast_ptr or 0)
                if mc and self.output == "fused-mc":
                    extra = Multicast(mc + 4 * self.lo)
                else:
                    extra = [int(handle.buffer_ptrs[r]) + 4 * self.lo for r in range(self.world) if r != self.rank]
                bufs.append((buf, handle, extra))
            self._symm = bufs
            self._calls = 0
        self._calls += 1
        return self._symm[self._calls % 2]

    def _stage_for(self, rows_local, dev):
        """Rows given as raw (possibly remote) addresses and read twice by a
        Krum-family rule (Gram, then combine): a local [n, d_local] staging
        matrix the Gram kernel fills on the way, or None."""
        from ._lib import DevicePtrRows
        if not isinstance(rows_local, DevicePtrRows) or not self._use_peer_exchange(dev):
            return None
        ld = (self.d_local + 3) // 4 * 4
        if getattr(self, "_stage", None) is None or self._stage.shape[1] < ld:
            self._stage = torch.empty((self.n, ld), dtype=torch.float32, device=dev)
        return self._stage

    def _use_peer_exchange(self, device, rows=None) -> bool:
        if self.world <= 1 or self.rule not in KRUM_FAMILY or device.type != "cuda":
            return False
        if rows is not None and is_bf16(rows):
            return False
        if self.exchange == "nccl" or not hasattr(self.backend, "gram_exchange"):
            return False
        return True

    def _exchange_buffers(self, device):
        """Symmetric buffer: two slot arrays fp64[world][n*n] (alternating per
        call) and the flag array uint32[world]; zeroed and fenced by a barrier
        once."""
        if self._xchg is None:
            import torch.distributed._symmetric_memory as symm_mem
            nn = self.n * self.n
            slot_bytes = self.world * nn * 8
            nbytes = 2 * slot_bytes + 4 * self.world + 16
            buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
            group = self.group if self.group is not None else dist.group.WORLD
            handle = symm_mem.rendezvous(buf, group)
            buf.zero_()
            handle.barrier()
            bases = [int(handle.buffer_ptrs[r]) for r in range(self.world)]
            self._xchg = {"buf": buf, "handle": handle, "bases": bases, "slot_bytes": slot_bytes, "epoch": 0}
        return self._xchg

    def _gram_whole(self, rows_local, dev, mark, stage=None):
        """Whole-vector Gram matrix on every rank (self._gram); with `stage`
        the Gram kernel also copies the rows there (fused ingress staging)."""
        if self._use_peer_exchange(dev, rows_local):
            x = self._exchange_buffers(dev)
            x["epoch"] += 1
            par = x["epoch"] % 2
            slots = [b + par * x["slot_bytes"] for b in x["bases"]]
            flags = [b + 2 * x["slot_bytes"] for b in x["bases"]]
            self.backend.gram_exchange(rows_local, self._gram, self._ws, self.d_local, slots, flags, self.rank,
                                       self.world, x["epoch"], stage=stage)
            mark("gram")
            mark("exchange")
            return
        self.backend.gram_partial(rows_local, self._gram, self._ws, self.d_local)
        mark("gram")
        if self.world > 1:
            dist.all_reduce(self._gram, op=dist.ReduceOp.SUM, group=self.group)
        mark("exchange")

    @property
    def fused_path(self) -> str | None:
        """"multicast" / "p2p" once the fused buffers exist, else None."""
        if self._symm is None:
            return None
        return "multicast" if isinstance(self._symm[0][2], Multicast) else "p2p"

    # -- lazily created per-device state ------------------------------------------
    def _state(self, device):
        if self.rule in KRUM_FAMILY:
            if self._gram is None:
                from . import _lib
                nbytes = max(_lib.gar_workspace_bytes(self.rule, self.n, self.f, self.d_local), 1) \
                    if device.type == "cuda" else 1
                self._ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
                self._gram = torch.empty((self.n, self.n), dtype=torch.float64, device=device)
                self._idx = torch.empty(64, dtype=torch.int32, device=device)
        elif self._agg is None and device.type == "cuda":
            from .gar import init
            self._agg = init(self.rule, self.n, self.f, self.m or None)

    def aggregate(self, rows_local, out_local: torch.Tensor | None = None,
                  out_full: torch.Tensor | None = None, mark=None, barrier: bool = True) -> torch.Tensor:
        """rows_local: [n, >= d_local] slice of the gradients.  Returns the
        local slice (output="sharded") or the whole aggregate (replicated).
        `mark(label)`, if given, is called after each stage ("gram",
        "exchange", "select", "combine", "coord", "gather") — the benchmark
        records CUDA events there.  Fused outputs: barrier=False skips the
        cross-GPU barrier that makes the replicated output readable; the
        caller then calls sync() (any aggregator of the group) before reading
        it, and reads it before its next sync()."""
        dev = rows_local.device if hasattr(rows_local, "device") else rows_local[0].device
        self._state(dev)
        mark = mark or (lambda label: None)
        if self.output in ("fused", "fused-mc") and self.world > 1:
            return self._aggregate_fused(rows_local, dev, mark, barrier)
        if out_local is None:
            out_local = torch.empty(self.d_local, dtype=torch.float32, device=dev)
        if self.rule in KRUM_FAMILY:
            stage = self._stage_for(rows_local, dev)
            self._gram_whole(rows_local, dev, mark, stage)
            self.backend.select_from_gram(self.rule, self._gram, self.n, self.f, self.m, self._idx, ws=self._ws)
            mark("select")
            self.backend.combine(self.rule, stage if stage is not None else rows_local, self.f, self.m, self._idx,
                                 out_local, self.d_local)
            mark("combine")
        else:
            self.backend.coordinatewise(self._agg, rows_local, out_local, self.d_local)
            mark("coord")
        if self.output == "sharded" or self.world == 1:
            return out_local
        if out_full is None:
            out_full = torch.empty(self.per * self.world, dtype=torch.float32, device=dev)
        src = out_local
        if self.d_local != self.per:
            if self._pad is None:
                self._pad = torch.zeros(self.per, dtype=torch.float32, device=dev)
            self._pad[: self.d_local].copy_(out_local)
            src = self._pad
        if self.output == "replicated-async":
            # the all-gather runs on NCCL's stream and overlaps whatever the
            # caller launches next; wait() before reading out_full
            self._pending = dist.all_gather_into_tensor(out_full, src, group=self.group, async_op=True)
        else:
            dist.all_gather_into_tensor(out_full, src, group=self.group)
        mark("gather")
        return out_full[: self.d]

    def wait(self):
        """Make the current stream wait for a pending "replicated-async" gather."""
        if getattr(self, "_pending", None) is not None:
            self._pending.wait()
            self._pending = None

    def sync(self):
        """Cross-GPU barrier of the fused output: after it, every output
        written by this group's earlier calls (on every rank) is readable."""
        if self._symm is not None:
            self._symm[0][1].barrier()

    def _aggregate_fused(self, rows_local, dev, mark, barrier=True):
        buf, handle, extra = self._fused_buffers(dev)
        out_local = buf[self.lo: self.hi]
        if self.rule in KRUM_FAMILY:
            stage = self._stage_for(rows_local, dev)
            self._gram_whole(rows_local, dev, mark, stage)
            self.backend.select_from_gram(self.rule, self._gram, self.n, self.f, self.m, self._idx, ws=self._ws)
            mark("select")
            self.backend.combine(self.rule, stage if stage is not None else rows_local, self.f, self.m, self._idx,
                                 out_local, self.d_local, extra)
            mark("combine")
        else:
            self.backend.coordinatewise_bcast(self._agg, rows_local, out_local, self.d_local, extra)
            mark("coord")
        if barrier:
            handle.barrier()    # every rank's slices have landed in every buffer
        mark("gather")
        return buf[: self.d]

    @property
    def selected(self) -> torch.Tensor | None:
        """Indices chosen by the last Krum-family call (device int32)."""
        if self._idx is None:
            return None
        from . import _lib
        return self._idx[: _lib.gar_num_selected(self.rule, self.n, self.f, self.m)]


class WorkerShards:
    """Worker-major input for the d-sharded GARs: in data
    parallelism each GPU holds the FULL gradients of its own workers (worker
    w lives on rank w mod world), while rank s aggregates coordinate slice s
    of every worker's gradient.  Instead of an all-to-all into the d-sharded
    layout, the gradients sit in one symmetric-memory buffer per rank and
    rank s's kernels read slice s of each remote worker's row in place over
    NVLink (their TMA bulk copies / loads take peer addresses), so the
    exchange is fused into the aggregation kernels and needs no extra
    memory.  fill local_rows(), call ready() on every rank, then pass
    slice_rows(lo) to ShardedAggregator.aggregate."""

    def __init__(self, n: int, d: int, group=None, device=None):
        import torch.distributed._symmetric_memory as symm_mem
        from ._lib import DevicePtrRows
        self._rows_cls = DevicePtrRows
        self.n, self.d = int(n), int(d)
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ld = (self.d + 3) // 4 * 4
        self.local_workers = [w for w in range(self.n) if w % self.world == self.rank]
        per_rank = (self.n + self.world - 1) // self.world
        self.buf = symm_mem.empty(per_rank * self.ld, dtype=torch.float32, device=self.device)
        self.handle = symm_mem.rendezvous(self.buf, self.group)
        self.bases = [int(self.handle.buffer_ptrs[r]) for r in range(self.world)]

    def local_rows(self) -> torch.Tensor:
        """[len(local_workers), ld] view: row j is worker local_workers[j]."""
        return self.buf[: len(self.local_workers) * self.ld].view(len(self.local_workers), self.ld)

    def ready(self):
        """Barrier: every rank's local rows are written and visible."""
        self.handle.barrier()

    def slice_rows(self, lo: int):
        """The n rows of coordinates [lo, ...) as raw addresses, worker order."""
        ptrs = [self.bases[w % self.world] + 4 * ((w // self.world) * self.ld + lo) for w in range(self.n)]
        return self._rows_cls(ptrs, self.device)
