#!/usr/bin/env python3
"""Benchmark of the Garfield GAR hot path on B200.

Metric (BASELINE.json): GAR throughput in GB/s of gradients, n*d*4 bytes per
rule / time, plus the dominant kernel's fraction of the HBM roofline.

A step is one pass of the whole hot path (every row of SURVEY.md §8(a)) over
the workload: Average, Median, trimmed mean, Krum, Multi-Krum and Bulyan, each
aggregating the same n resident gradients.  Default workload = BASELINE.json
configs[2] (ResNet-50-sized gradients, n=31, f=7, d=25,557,032: the config the
north_star targets and scales to 8 GPUs); inputs (3.17 GB) exceed the 126 MB
L2, so no flush is needed between steps.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--dtype bf16]
    torchrun --nproc-per-node N bench.py --gpus N ...   (d-sharded, NCCL)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")
KRUM = ("krum", "multi_krum", "bulyan")
METRIC = "GAR throughput GB/s of gradients (n*d*4B/time), all six GARs per step"
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3", help="C1..C4 or sweep:<n>")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="auto", choices=["auto", "peer", "nccl"],
                    help="N>1 Krum-family Gram exchange: peer-memory kernels (auto/peer) or NCCL all-reduce")
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"],
                    help="element type of the gradients (bf16: SURVEY §8f-4, widened exactly, DESIGN.md R16)")
    ap.add_argument("--no-variants", action="store_true",
                    help="skip the bf16 variant measured after the fp32 line's timed region (N=1)")
    ap.add_argument("--output", default="sharded",
                    choices=["replicated", "replicated-async", "sharded", "fused", "fused-mc"],
                    help="N>1: keep the aggregate d-sharded (the primary number, SURVEY.md §8e: a ZeRO-style "
                         "consumer updates its own parameter shard), all-gather it to every rank with NCCL, or "
                         "write it into every rank's buffer from the producing kernel over NVLink (fused); with "
                         "sharded, the fused replicated output is measured after the timed region as a variant")
    return ap.parse_args()


def workload(name):
    if name.startswith("sweep:"):
        return synth.sweep_config(int(name.split(":")[1]))
    return synth.CONFIGS[name]


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def rule_bytes(rule, n, f, d, es=4):
    """Algorithmic HBM bytes of one aggregation: input rows of
    es bytes per coordinate read, the fp32 output written."""
    if rule in ("average", "median", "trimmed_mean"):
        return es * d * n + 4 * d
    if rule == "krum":
        return es * d * (n + 1) + 4 * d
    if rule == "multi_krum":
        return es * d * (n + (n - f - 2)) + 4 * d
    return es * d * (n + (n - 2 * f)) + 4 * d


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line):
    ONE process per node (local rank 0) querying every GPU every 200 ms, started
    before the ranks' pre-timing barrier (profiles/r2_multigpu.md: starting a
    sampler between the barrier and t0 skewed the ranks by nvidia-smi's start-up
    time, which the earliest rank then timed at its first cross-rank sync)."""

    def __init__(self, index, active=True):
        self.index = index
        self.active = active
        self.proc = None
        self.path = None

    def __enter__(self):
        if not self.active:
            return self
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            if os.environ.get("GAR_BENCH_NO_SMI"):         # diagnostics only: no sampler
                raise RuntimeError("sampler disabled")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        # the sampler must be running before the timed region starts: wait for
        # its first lines (nvidia-smi can take a second to start on a cold box)
        t_end = time.time() + 5.0
        while self.proc is not None and time.time() < t_end:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.05)
        self._lines0 = self._count()
        return self

    def _count(self):
        try:
            with open(self.path) as fh:
                return sum(1 for _ in fh)
        except (OSError, TypeError):
            return 0

    def __exit__(self, *a):
        # keep sampling until one more round of samples covers the timed region
        t_end = time.time() + 2.0
        while self.proc is not None and self._count() <= self._lines0 and time.time() < t_end:
            time.sleep(0.05)
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self, gpus=None):
        """Median SM clock under load, max clock and throttle reasons over the
        job's GPUs (indices `gpus`, default all sampled)."""
        if not self.active:
            return None
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines()]
            rows = [[c.strip() for c in r] for r in rows if len(r) >= 9]
            if gpus is not None:
                rows = [r for r in rows if int(r[0]) in gpus]
            sm = [float(r[1]) for r in rows]
            mx = max(float(r[2]) for r in rows)
            reasons = set()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in rows:
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(rows)}
        except Exception as e:  # pragma: no cover
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)}
        finally:
            try:
                os.remove(self.path)
            except OSError:
                pass


def traffic_from_profiles(kernel, workload, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`,
    from the committed `ncu --set full` capture of the default single-GPU C3
    step (profiles/traffic.json, written by tools/summarize_ncu.py); other
    configurations report null."""
    if workload != "C3" or world != 1:
        return None
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        base = kernel.split("<")[0]
        for k, v in t.get("per_kernel", {}).items():   # ncu names carry a namespace prefix
            if k.split("::")[-1].split("<")[0] == base:
                return v
        return None
    except Exception:
        return None


# ============================================================== our implementation
def run_ours(args):
    import torch
    import torch.distributed as dist

    import __graft_entry__
    # compile libgar.so in-tree if missing or stale (clean checkout), outside
    # any timed region; concurrent ranks serialise on the builder's lock
    __graft_entry__.ensure_built(with_oracle=False)
    import paper_2010_05888_b200 as gar  # noqa: F401

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workload(args.workload)
    n, f, d = cfg.n, cfg.f, cfg.d
    lo, hi = synth.shard_bounds(d, rank, world) if world > 1 else (0, d)
    dl = hi - lo
    X = synth.make_gradients(n, f, dl, seed=synth.BASE_SEED + 2 + 1000 * rank, device=dev)
    bf16 = args.dtype == "bf16"
    if bf16:
        X = synth.to_bf16(X)
        if world > 1 and args.output not in ("replicated", "sharded"):
            args.output = "replicated"          # fused outputs take fp32 rows (dist._LibgarBackend)
    es = X.element_size()
    torch.cuda.synchronize()

    from paper_2010_05888_b200.dist import ShardedAggregator, shard_len
    aggs = {r: ShardedAggregator(r, n, f, d, output=args.output, exchange=args.exchange) for r in RULES}
    outs = {r: torch.empty(dl, dtype=torch.float32, device=dev) for r in RULES}
    full = {r: torch.empty(shard_len(d, world) * world, dtype=torch.float32, device=dev) for r in RULES} \
        if world > 1 else {r: None for r in RULES}
    stream = torch.cuda.current_stream(dev)
    # kernel class of the stage ending at each mark (DESIGN.md §8 roofline bookkeeping)
    CLASS = {"gram": "gram", "exchange": "exchange", "select": "select", "combine": "coord_select",
             "coord": "coord_select", "gather": "gather"}

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def step(Xin, segs, A=None):
        # fused output: one cross-GPU barrier per step (the last rule's), which
        # makes all six replicated outputs readable (dist.ShardedAggregator.sync)
        A = A or aggs
        for r in RULES:
            last_rule = r == RULES[-1]
            if segs is None:
                A[r].aggregate(Xin, out_local=outs[r], out_full=full[r], barrier=last_rule)
                continue
            last = [ev()]

            def mark(label, r=r, last=last):
                e = ev()
                segs.append((label, r, last[0], e))
                last[0] = e
            A[r].aggregate(Xin, out_local=outs[r], out_full=full[r], mark=mark, barrier=last_rule)
        for r in RULES:              # output="replicated-async": the step ends when every gather has
            A[r].wait()              # landed (they overlap the following rules' kernels)

    def measure(Xin, steps, warmup, clocks=True, A=None):
        """(ms over `steps` steps, segments, clock summary), max over ranks."""
        segs = []
        for _ in range(warmup):
            step(Xin, None, A)
        torch.cuda.synchronize()
        # the sampler starts (and delivers its first sample) BEFORE the ranks'
        # barrier: a rank that entered the timed region while another still
        # waited for nvidia-smi would time that wait at its first cross-rank sync
        with Clocks(local, active=(local == 0)) as clk:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = ev()
            for _ in range(steps):
                step(Xin, segs, A)
            t1 = ev()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # the job's GPUs: cuda:0..N-1 are nvidia-smi indices 0..N-1 unless remapped
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        gpus = set(range(world)) if not vis else {int(v) for v in vis.split(",")[:world] if v.strip().isdigit()}
        return t0.elapsed_time(t1), segs, clk.summary(gpus or None)

    def rule_times(segs):
        cls_ms, rule_ms = {}, {r: 0.0 for r in RULES}
        for lab, r, a, b in segs:
            t = a.elapsed_time(b)
            cls_ms[CLASS[lab]] = cls_ms.get(CLASS[lab], 0.0) + t
            rule_ms[r] += t
        return cls_ms, rule_ms

    ms, segs, clocks = measure(X, args.steps, args.warmup)
    cls_ms, rule_ms = rule_times(segs)
    if os.environ.get("GAR_BENCH_PER_RANK"):    # diagnostics: this rank's own times (stderr)
        print(json.dumps({"rank": rank, "ms_per_step": round(ms / args.steps, 4),
                          "per_rule": {r: round(t / args.steps, 4) for r, t in rule_ms.items()},
                          "stages": {c: round(t / args.steps, 4) for c, t in cls_ms.items()}}),
              file=sys.stderr, flush=True)
    if world > 1:
        t = torch.tensor([ms] + [rule_ms[r] for r in RULES], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        rule_ms = {r: float(t[1 + i]) for i, r in enumerate(RULES)}

    # ---- e2e through the public API with host buffers (pinned), copies in the timed region.
    # Every step copies its inputs host -> device and its six results device ->
    # host.  Copies run on their own streams and the input / output buffers are
    # double-buffered, so step k+1's H2D overlaps step k's aggregation and D2H.
    e2e = None
    if args.e2e_steps > 0:
        host_x = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
        host_x.copy_(X)
        host_out = [{r: torch.empty(dl, dtype=torch.float32, pin_memory=True) for r in RULES} for _ in range(2)]
        xbuf = [X, torch.empty_like(X)]
        obuf = [outs, {r: torch.empty(dl, dtype=torch.float32, device=dev) for r in RULES}]
        fbuf = [full, {r: (torch.empty_like(full[r]) if full[r] is not None else None) for r in RULES}]
        h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        pub = {r: gar.init(r, n, f) for r in RULES}
        for r in RULES:                            # workspace allocation outside the timed region
            pub[r].aggregate(X, out=outs[r], d=dl)
        consumed = [None, None]                    # compute finished reading xbuf[b]
        drained = [None, None]                     # D2H finished reading obuf[b]
        rule_drained = {}
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = ev()
        h2d.wait_event(a)
        d2h.wait_event(a)
        for k in range(args.e2e_steps):
            bb = k % 2
            with torch.cuda.stream(h2d):
                if consumed[bb] is not None:
                    h2d.wait_event(consumed[bb])
                xbuf[bb].copy_(host_x, non_blocking=True)
                loaded = torch.cuda.Event()
                loaded.record(h2d)
            stream.wait_event(loaded)
            if drained[bb] is not None:
                stream.wait_event(drained[bb])
            for r in RULES:
                if r in rule_drained:              # fused outputs live in the aggregator's own buffer
                    stream.wait_event(rule_drained[r])
                if world == 1:         # the public single-GPU call: Aggregator.aggregate -> gar_aggregate_ex
                    res = pub[r].aggregate(xbuf[bb], out=obuf[bb][r], d=dl)
                else:                  # the public multi-GPU call (Aggregator.aggregate_sharded's engine)
                    res = aggs[r].aggregate(xbuf[bb], out_local=obuf[bb][r], out_full=fbuf[bb][r],
                                            barrier=r == RULES[-1])
                    aggs[r].wait()
                local_res = res[lo:hi] if res.numel() > dl else res
                done = torch.cuda.Event()
                done.record(stream)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(done)
                    host_out[bb][r].copy_(local_res, non_blocking=True)
                    rule_drained[r] = torch.cuda.Event()
                    rule_drained[r].record(d2h)
            consumed[bb] = torch.cuda.Event()
            consumed[bb].record(stream)
            drained[bb] = torch.cuda.Event()
            drained[bb].record(d2h)
        stream.wait_stream(h2d)
        stream.wait_stream(d2h)
        b = ev()
        torch.cuda.synchronize()
        e2e_ms = a.elapsed_time(b) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t[0])
        del xbuf[1], fbuf[1]
        e2e = {"value": round(len(RULES) * n * d * es / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": int(X.numel() * es * world),
               "d2h_bytes_per_step": int(len(RULES) * dl * 4 * world),
               "path": ("paper_2010_05888_b200.init(rule, n, f).aggregate(X) per rule (one "
                        + ("gar_aggregate_dt" if bf16 else "gar_aggregate_ex") + " C call each)" if world == 1 else
                        "dist.ShardedAggregator.aggregate per rule (gar_gram_exchange / gar_select_from_gram / "
                        "gar_combine_bcast for the Krum family, gar_aggregate_bcast otherwise)")
                       + "; inputs H2D from pinned host and six results D2H every step, on copy streams, "
                         "double-buffered so step k+1's H2D overlaps step k's aggregation"}

    # ---- the bf16 variant of the same workload, after the
    # timed region of the line: same bits rounded to bf16, same step
    variant = None
    if world == 1 and not bf16 and not args.no_variants:
        X16 = synth.to_bf16(X)
        ms16, segs16, clk16 = measure(X16, args.steps, max(args.warmup, 3))
        del X16
    # ---- N > 1 with the sharded output: the replicated output (every rank
    # receives the whole aggregate, written by the producing kernels over
    # NVLink) on the same step, after the timed region (both reported)
    rep_ms = None
    if world > 1 and args.output == "sharded" and not args.no_variants:
        rep_out = "fused" if not bf16 else "replicated"
        rep = {r: ShardedAggregator(r, n, f, d, output=rep_out, exchange=args.exchange) for r in RULES}
        rep_ms, _, rep_clk = measure(X, args.steps, max(args.warmup, 3), A=rep)
        t = torch.tensor([rep_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rep_ms = float(t[0])
        rep_path = rep[RULES[0]].fused_path
        del rep
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_src = peaks()
    m_mk, theta = n - f - 2, n - 2 * f
    np_ = 8 if n <= 8 else 16 if n <= 16 else 32 if n <= 32 else 64

    def kernel_table(segs, ms_step, esz):
        """Per-kernel roofline: every timed segment is one
        libgar kernel launch, except "gram", which is the Gram kernel plus the
        deterministic n x n partial reduction (~1 % of it; counted against the
        Gram, so its fraction is conservative).  Algorithmic bytes per launch on
        this rank's slice: rows read (esz bytes per coordinate) + fp32 output."""
        kern = {}

        def add(name, t_ms, nbytes):
            k = kern.setdefault(name, {"ms_per_step": 0.0, "launches_per_step": 0, "bytes": 0})
            k["ms_per_step"] += t_ms / args.steps
            k["launches_per_step"] += 1
            k["bytes"] += nbytes
        seg_name = {"krum": ("copy_row_kernel", (esz + 4) * dl),
                    "multi_krum": ("coord_select_kernel<average of m selected rows>", (esz * m_mk + 4) * dl),
                    "bulyan": ("coord_select_kernel<bulyan coordinate phase>", (esz * theta + 4) * dl)}
        for lab, r, a, b in segs:
            t = a.elapsed_time(b)
            if lab == "gram":
                add(f"gram_tc_kernel<{np_}>", t, esz * n * dl)
            elif lab == "select":
                add("select_kernel", t, 0)
            elif lab == "combine":
                add(seg_name[r][0], t, seg_name[r][1])
            elif lab == "coord":
                add(f"coord_select_kernel<{r}>", t, (esz * n + 4) * dl)
        reps = args.steps   # every segment was recorded once per rule per step
        kernels = {}
        for name, k in kern.items():
            per_launch_ms = k["ms_per_step"] * reps / k["launches_per_step"]     # average launch duration
            per_launch_bytes = k["bytes"] / k["launches_per_step"]
            ach = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 and per_launch_bytes else 0.0
            kernels[name] = {"ms_per_step": round(k["ms_per_step"], 4),
                             "launches_per_step": k["launches_per_step"] // reps,
                             "ms_per_launch": round(per_launch_ms, 4),
                             "algorithmic_bytes_per_launch": int(per_launch_bytes),
                             "achieved_gbs": round(ach, 1), "frac": round(ach / peak, 4) if ach else None,
                             "share_of_step": round(k["ms_per_step"] / ms_step, 4)}
        return kernels

    def per_rule_table(rms, esz):
        out = {}
        for r in RULES:
            t = rms[r] / args.steps
            out[r] = {"ms": round(t, 4), "grad_gbs": round(n * d * esz / (t * 1e-3) / 1e9, 1),
                      "roofline_frac": round(rule_bytes(r, n, f, d, esz) / world / (t * 1e-3) / 1e9 / peak, 4)}
        return out

    ms_step = ms / args.steps
    grad_bytes = len(RULES) * n * d * es
    value = grad_bytes / (ms_step * 1e-3) / 1e9
    kernels = kernel_table(segs, ms_step, es)
    dom = max((k for k in kernels if kernels[k]["algorithmic_bytes_per_launch"]),
              key=lambda k: kernels[k]["ms_per_step"])
    # libgar kernels per step: 1 per coordinate-wise rule; per Krum-family rule
    # Gram partials + reduction + selection + combine, and with the peer-memory
    # exchange (N > 1) the reduction is a reduce-and-store plus a gather kernel
    peer = world > 1 and aggs["krum"]._use_peer_exchange(dev, X)
    launches_per_step = 3 + 3 * (5 if peer else 4)
    stages = {c: round(t / args.steps, 4) for c, t in sorted(cls_ms.items())}
    per_rule = per_rule_table(rule_ms, es)
    if rep_ms is not None:
        variant = {"replicated_output": {
            "what": "the same step with the aggregate replicated on every rank (output=" + rep_out
                    + (f" ({rep_path})" if rep_path else "") + "), measured after this line's timed region",
            "value": round(grad_bytes / (rep_ms / args.steps * 1e-3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(rep_ms / args.steps, 4), "clocks": rep_clk}}
    if world == 1 and not bf16 and not args.no_variants:
        ms16_step = ms16 / args.steps
        k16 = kernel_table(segs16, ms16_step, 2)
        variant = {"bf16": {
            "what": "the same step on the same gradients rounded to bf16 (gar_*_dt, exact widening, DESIGN.md R16), "
                    "measured after this line's timed region; gradient bytes n*d*2",
            "value": round(len(RULES) * n * d * 2 / (ms16_step * 1e-3) / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(ms16_step, 4), "speedup_vs_f32": round(ms_step / ms16_step, 3),
            "per_rule": per_rule_table(rule_times(segs16)[1], 2), "kernels": k16, "clocks": clk16}}
    metric = METRIC if not bf16 else METRIC.replace("n*d*4B", "n*d*2B bf16")
    line = {
        "metric": metric, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16" if bf16 else "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name}: n={n} f={f} d={d}, GARs {'/'.join(RULES)}",
                   "n": n, "f": f, "d": d, "parallelism": f"d-sharded x{world}" if world > 1 else "single GPU",
                   "output": (args.output + (f" ({aggs[RULES[0]].fused_path})" if aggs[RULES[0]].fused_path else ""))
                   if world > 1 else "local",
                   "l2": f"inputs {n * d * es / 1e9:.2f} GB > 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": kernels[dom]["achieved_gbs"], "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": kernels[dom]["frac"],
                     "algorithmic_bytes_per_launch": kernels[dom]["algorithmic_bytes_per_launch"],
                     "launches_per_step": kernels[dom]["launches_per_step"],
                     "share_of_step": kernels[dom]["share_of_step"],
                     "traffic": traffic_from_profiles(dom, args.workload, world) if not bf16 else None},
        "kernels": kernels, "per_rule": per_rule, "clocks": clocks,
        "stages_ms": stages, "gpu_launches": launches_per_step * args.steps, "e2e": e2e,
    }
    if variant:
        line["variants"] = variant
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, X, d)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ============================================================== the oracle as the reference arm
def oracle_step(x, f):
    import oracle
    for r in RULES:
        oracle.aggregate(r, x, f)


def cpu_baseline(cfg, X, d, reps=3):
    """The oracle, as it stands, on the box's host cores over the SAME resident
    workload (copied to host; bf16 rows widened exactly first, R16): all six
    GARs once per repetition, median of `reps` (about 10-30 s of CPU work at C3)."""
    import oracle
    import torch
    if X.dtype == torch.bfloat16:
        x = oracle.widen_bf16(synth.bf16_bits(X[:, :d]))
    else:
        x = X[:, :d].cpu().numpy()
    x = x if x.flags["C_CONTIGUOUS"] else x.copy()
    times = []
    for _ in range(reps):
        t = time.perf_counter()
        oracle_step(x, cfg.f)
        times.append(time.perf_counter() - t)
    dt = statistics.median(times)
    return {"value": round(len(RULES) * cfg.n * d * 4 / dt / 1e9, 4), "unit": "GB/s",
            "cores": oracle.default_threads(), "kind": "oracle",
            "sample": f"the full {cfg.name} workload (n={cfg.n} f={cfg.f} d={d}, same bits as the GPU run), "
                      f"all six GARs, median of {reps} passes ({dt:.2f} s per pass)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cfg = workload(args.workload)
    sample_d = min(1 << 21, cfg.d)
    x = synth.make_gradients(cfg.n, cfg.f, sample_d, seed=synth.BASE_SEED + 2, ld=sample_d).numpy()
    for _ in range(args.warmup):
        oracle_step(x, cfg.f)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(x, cfg.f)
    dt = (time.perf_counter() - t) / args.steps
    value = len(RULES) * cfg.n * sample_d * 4 / dt / 1e9
    part = f"first {sample_d} of {cfg.d} coordinates" if sample_d < cfg.d else f"all {cfg.d} coordinates"
    sample = f"{cfg.name} shape n={cfg.n} f={cfg.f}, {part} per step, all six GARs"
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: n={cfg.n} f={cfg.f} d={cfg.d}, GARs {'/'.join(RULES)}",
                       "n": cfg.n, "f": cfg.f, "d": cfg.d,
                       "sample": f"each step aggregates the {part} (value = gradient bytes of the sample / time)"},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": oracle.default_threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
