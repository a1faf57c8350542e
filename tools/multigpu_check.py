"""torchrun target of tests/test_multigpu_gpu.py: the d-sharded path on real
GPUs (one process per GPU, NCCL + symmetric memory) against the ORACLE on the
whole vectors.

Every rank generates the same whole [n, d] matrix (seeded, well-separated
selections) and aggregates its coordinate slice through
dist.ShardedAggregator in every output mode / exchange; rank 0 checks the
replicated outputs bit for bit against the oracle's aggregate of the whole
vectors and the selections exactly against the oracle's; every rank checks its
outputs equal rank 0's (all-gathered).  bf16 rows: the NCCL exchange with a
replicated output.  Prints one line "multigpu check: ok" or raises."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2010_05888_b200.dist import ShardedAggregator, shard_bounds  # noqa: E402

RULES = ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan", "mda", "mean_around_median")
MODES = (("replicated", "nccl"), ("replicated", "peer"), ("fused", "peer"), ("fused-mc", "peer"),
         ("sharded", "peer"))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    n, f, d = 19, 4, 1_000_003
    Xw = synth.make_gradients(n, f, d, seed=4242, kind="separated", device=dev)   # same bits on every rank
    lo, hi = shard_bounds(d, rank, world)
    Xl = torch.zeros((n, synth.aligned_ld(hi - lo)), dtype=torch.float32, device=dev)   # 16-byte aligned rows
    Xl[:, : hi - lo] = Xw[:, lo:hi]
    x_host = Xw[:, :d].cpu().numpy() if rank == 0 else None
    D = None
    if rank == 0:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        import oracle
        D = oracle.distances(x_host)
    checked = 0
    for dtype in (torch.float32, torch.bfloat16):
        rows = Xl if dtype == torch.float32 else synth.to_bf16(Xl)
        xd = None
        if dtype == torch.bfloat16 and rank == 0:
            import oracle
            xd = np.ascontiguousarray(oracle.widen_bf16(synth.bf16_bits(synth.to_bf16(Xw[:, :d]))[:, :d]))
            Dxd = oracle.distances(xd)
        for rule in RULES:
            ff = 2 if rule == "mda" else f
            modes = MODES if dtype == torch.float32 else (("replicated", "nccl"), ("sharded", "nccl"))
            for output, exch in modes:
                agg = ShardedAggregator(rule, n, ff, d, output=output, exchange=exch)
                for _ in range(2):
                    out = agg.aggregate(rows)
                if output == "sharded":
                    full = torch.empty(agg.per * world, dtype=torch.float32, device=dev)
                    pad = torch.zeros(agg.per, dtype=torch.float32, device=dev)
                    pad[: hi - lo].copy_(out[: hi - lo])
                    dist.all_gather_into_tensor(full, pad)
                    out = torch.cat([full[r * agg.per: r * agg.per + (shard_bounds(d, r, world)[1] -
                                                                      shard_bounds(d, r, world)[0])]
                                     for r in range(world)])
                torch.cuda.synchronize()
                got = out[:d].cpu().numpy()
                sel = agg.selected.cpu().numpy() if agg.selected is not None else None
                # every rank holds the same result as rank 0
                mine = torch.from_numpy(got.view(np.int32)).to(dev)
                r0 = mine.clone()
                dist.broadcast(r0, 0)
                if not torch.equal(mine, r0):
                    raise AssertionError(f"rank {rank}: {rule} {output}/{exch} {dtype} differs from rank 0")
                if rank == 0:
                    import oracle
                    from gpu_helpers import assert_same_bits, assert_selection
                    xx = x_host if dtype == torch.float32 else xd
                    what = f"{rule} {output}/{exch} {dtype} world={world}"
                    if rule in ("average", "median", "trimmed_mean"):
                        exp = oracle.aggregate(rule, xx, f)[0]
                    elif rule == "mean_around_median":
                        exp = oracle.mean_around_median(xx, f)
                    else:
                        Dx = D if dtype == torch.float32 else Dxd
                        if rule == "mda":
                            rsel = oracle.mda_select(Dx, 2)
                            if list(sel) != list(rsel):
                                diam = lambda s_: max((Dx[i, j] for i in s_ for j in s_ if i < j), default=0.0)
                                assert diam(sel) <= diam(rsel) * (1 + 1e-5), (what, list(sel), list(rsel))
                        else:
                            assert_selection(rule, Dx, f, 1 if rule == "krum" else n - f - 2, sel)
                        exp = oracle.bulyan_coordinate_phase(xx, f, sel) if rule == "bulyan" else \
                            oracle.mean_of_rows(xx, sel)
                    assert_same_bits(got, exp, what)
                checked += 1
    dist.barrier()
    if rank == 0:
        print(f"multigpu check: ok ({checked} cases, world {world})", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
