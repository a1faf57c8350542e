"""The default multi-GPU path ("GPU-to-GPU
communication") on ONE GPU: W fake ranks, each with its own CUDA stream,
slot array and flag array in this GPU's memory, run exactly the calls
dist.ShardedAggregator makes per rank for output="fused":

  Krum family:  gar_gram_exchange (Gram partials over the rank's coordinate
                slice + peer-memory reduce / flag handshake / rank-order sum)
                -> gar_select_from_gram -> gar_combine_bcast (the rank's output
                slice stored into every rank's replicated buffer);
  coordinate-wise: gar_aggregate_bcast.

Checked: every rank holds the bit-identical Gram matrix, equal to the sum in
rank order of per-slice gar_gram_partial matrices; the selection equals the
ORACLE's on the whole vectors (exact: the input is well separated); every
rank's replicated output is bitwise equal to the single-call result on the
whole vectors.  Sizes keep all fake ranks' kernels co-resident on the GPU
(<= 64 Gram CTAs per rank), since a real rank's spin-wait never shares an SM
with another rank's Gram.  Every kernel is launched once (a world = 1 pass)
before the fake ranks run: with CUDA's lazy module loading, the first launch
of a kernel blocks the host thread while a fake rank's kernel spin-waits for
a rank that this same thread has not launched yet."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_helpers import KRUM_FAMILY, assert_same_bits, assert_selection, to_device

pytestmark = pytest.mark.gpu

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")


@pytest.fixture(scope="module")
def gar():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2010_05888_b200 as g
    return g


@pytest.mark.parametrize("world,n,f,d", [(2, 31, 7, 16_001), (4, 31, 7, 16_387), (2, 11, 2, 9_001),
                                         (3, 63, 15, 12_289), (8, 19, 4, 30_000)])
def test_fake_ranks_exchange_and_fused_output(gar, world, n, f, d):
    x = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 31 * world + n, ld=d, kind="separated").numpy()
    X = to_device(x)
    dev = X.device
    bounds = [synth.shard_bounds(d, r, world) for r in range(world)]
    per = bounds[0][1] - bounds[0][0]
    streams = [torch.cuda.Stream(dev) for _ in range(world)]
    D = oracle.distances(x)
    ws = [torch.empty(gar.gar_workspace_bytes("bulyan", n, f, d), dtype=torch.uint8, device=dev)
          for _ in range(world)]
    _run_fake_ranks(gar, X, n, f, d, [(0, d)], 1, ws, [torch.cuda.current_stream(dev)], D=None, x=None)
    _run_fake_ranks(gar, X, n, f, d, bounds, world, ws, streams, D=D, x=x)


def _run_fake_ranks(gar, X, n, f, d, bounds, world, ws, streams, D, x):
    dev = X.device
    per = bounds[0][1] - bounds[0][0]
    for epoch, rule in enumerate(RULES, start=1):
        # per-rank symmetric state (what dist.ShardedAggregator allocates in symmetric memory)
        slots = [torch.zeros(world * n * n, dtype=torch.float64, device=dev) for _ in range(world)]
        flags = [torch.zeros(world, dtype=torch.int32, device=dev) for _ in range(world)]
        full = [torch.full((per * world,), float("nan"), dtype=torch.float32, device=dev) for _ in range(world)]
        grams = [torch.empty((n, n), dtype=torch.float64, device=dev) for _ in range(world)]
        idx = [torch.full((64,), -1, dtype=torch.int32, device=dev) for _ in range(world)]
        torch.cuda.synchronize()
        for r, (lo, hi) in enumerate(bounds):
            rows = [X[i, lo:hi] for i in range(n)]
            extra = [full[q].data_ptr() + 4 * lo for q in range(world) if q != r]
            out_local = full[r][lo:hi]
            with torch.cuda.stream(streams[r]):
                if rule in KRUM_FAMILY:
                    gar.gar_gram_exchange(rows, grams[r], ws[r], [s.data_ptr() for s in slots],
                                          [fl.data_ptr() for fl in flags], r, world, epoch, d=hi - lo)
                    gar.gar_select_from_gram(rule, grams[r], n, f, 0, idx[r], workspace=ws[r])
                    gar.gar_combine_bcast(rule, rows, f, 0, idx[r], out_local, extra, d=hi - lo)
                else:
                    gar.gar_aggregate_bcast(rule, rows, f, 0, out_local, extra, d=hi - lo)
        torch.cuda.synchronize()
        if D is None:          # the kernel warm-up pass
            continue
        # the single-call result on the whole vectors
        agg = gar.init(rule, n, f)
        one_idx = torch.full((64,), -1, dtype=torch.int32, device=dev)
        whole = agg.aggregate(X, d=d, indices=one_idx if rule in KRUM_FAMILY else None)
        torch.cuda.synchronize()
        for r in range(world):
            assert_same_bits(full[r][:d].cpu().numpy(), whole.cpu().numpy(), f"{rule} rank {r} replicated output")
        if rule in KRUM_FAMILY:
            # bit-identical Gram on every rank == per-slice partial Grams summed in rank order
            ref = torch.zeros((n, n), dtype=torch.float64, device=dev)
            for lo, hi in bounds:
                g = torch.empty((n, n), dtype=torch.float64, device=dev)
                gar.gar_gram_partial([X[i, lo:hi] for i in range(n)], g, ws[0], d=hi - lo)
                ref += g
            torch.cuda.synchronize()
            for r in range(world):
                assert torch.equal(grams[r], grams[0]), f"{rule}: rank {r} Gram differs from rank 0"
                assert torch.equal(idx[r], idx[0])
                assert int(flags[r].min()) == epoch
            assert torch.equal(grams[0], ref), f"{rule}: exchanged Gram != rank-order sum of slice partials"
            k = agg.num_selected
            sel = idx[0][:k].cpu().numpy()
            mm = 1 if rule == "krum" else n - f - 2
            assert assert_selection(rule, D, f, mm, sel, require_separated=True) == "exact"
            assert sel.tolist() == one_idx[:k].cpu().tolist()
        else:
            ref_o, _ = oracle.aggregate(rule, x, f)
            assert_same_bits(full[0][:d].cpu().numpy(), ref_o, f"{rule} vs oracle")
