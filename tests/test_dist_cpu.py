"""The d-sharded path's host logic over a real 2-rank gloo process group on CPU:
shard bounds, the partial-Gram all-reduce, identical selection on every rank,
per-slice combine and the output all-gather (padding of the last slice).  The
GPU kernels are replaced by a host test double (numpy / oracle); the result
must equal the oracle run on the whole, unsharded vectors."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_05888_b200.dist import ShardedAggregator, shard_bounds, shard_len

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan")


class HostBackend:
    """Test double with libgar's contract: gram_partial writes the Gram matrix
    of the (uncentred) slice; selection / combine follow the oracle."""

    def coordinatewise(self, agg, rows, out, d):
        import oracle
        x = rows[:, :d].numpy()
        res = {"average": lambda: oracle.average(x), "median": lambda: oracle.median(x, self.f),
               "trimmed_mean": lambda: oracle.trimmed_mean(x, self.f)}[self.rule]()
        out.copy_(torch.from_numpy(res))

    def gram_partial(self, rows, gram, ws, d):
        x = rows[:, :d].numpy().astype(np.float64)
        gram.copy_(torch.from_numpy(x @ x.T))

    def select_from_gram(self, rule, gram, n, f, m, idx, ws=None):
        import oracle
        G = gram.numpy()
        g = np.diag(G)
        D = g[:, None] + g[None, :] - 2 * G
        np.fill_diagonal(D, 0.0)
        if rule == "bulyan":
            sel = oracle.bulyan_select(D, f)
        else:
            sel = oracle.multi_krum_select(D, f, 1 if rule == "krum" else (m or n - f - 2))
        idx[: len(sel)] = torch.from_numpy(sel.astype(np.int32))
        return len(sel)

    def combine(self, rule, rows, f, m, idx, out, d):
        import oracle
        x = rows[:, :d].numpy()
        n = x.shape[0]
        k = n - 2 * f if rule == "bulyan" else (1 if rule == "krum" else (m or n - f - 2))
        sel = idx[:k].numpy()
        res = oracle.bulyan_coordinate_phase(x, f, sel) if rule == "bulyan" else oracle.mean_of_rows(x, sel)
        out.copy_(torch.from_numpy(res))


def _worker(rank, world, port, x, f, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n, d = x.shape
    lo, hi = shard_bounds(d, rank, world)
    local = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi]))
    out = {}
    for rule in RULES:
        be = HostBackend()
        be.rule, be.f = rule, f
        agg = ShardedAggregator(rule, n, f, d, backend=be)
        assert (agg.lo, agg.hi) == (lo, hi)
        full = agg.aggregate(local)
        out[rule] = (full.numpy().copy(), None if agg.selected is None else agg.selected.numpy().copy())
        agg_async = ShardedAggregator(rule, n, f, d, backend=be, output="replicated-async")
        full_async = agg_async.aggregate(local)
        agg_async.wait()
        assert np.array_equal(full_async.numpy(), out[rule][0])
    results[rank] = out
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("d", [5000, 3 * 1024 + 17])
def test_sharded_equals_whole_over_gloo(d):
    import oracle
    import synth
    n, f = 11, 2
    x = synth.make_gradients(n, f, d, seed=7, ld=d).numpy()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), x, f, results), nprocs=2, join=True)
    for rule in RULES:
        a, sa = results[0][rule]
        b, sb = results[1][rule]
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))      # identical on all ranks
        ref, sel = oracle.aggregate(rule, x, f)
        if sel is not None:
            assert sa.tolist() == sb.tolist() == sel.tolist(), rule
        np.testing.assert_array_equal(a.view(np.uint32), ref.view(np.uint32), rule)


def test_shard_bounds_cover_and_align():
    for d in (1, 1023, 1024, 25_557_032, 138_357_544):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(d, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == d
            for (a, b), (c, e) in zip(spans, spans[1:]):
                assert b == c
            per = shard_len(d, world)
            for r, (a, b) in enumerate(spans):
                assert a == min(d, r * per)
                if world > 1:
                    assert a % 1024 == 0 or a == d
