"""torchrun check: the fused output all-gather (symmetric memory; multicast
gar_*_mcast and peer-store gar_*_bcast) gives bit-identical replicated outputs
to the NCCL all-gather path, on every rank."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import synth
from paper_2010_05888_b200.dist import ShardedAggregator, shard_bounds

local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
n, f, d = 31, 7, 5_000_011
lo, hi = shard_bounds(d, rank, world)
X = synth.make_gradients(n, f, hi - lo, seed=11 + rank, device=dev)
bad = 0
for rule in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan", "mda", "mean_around_median"):
    a = ShardedAggregator(rule, n, f, d, output="replicated", exchange="nccl").aggregate(X).clone()
    for mode, exch in (("replicated", "peer"), ("fused", "peer"), ("fused", "nccl"), ("fused-mc", "peer")):
        fu = ShardedAggregator(rule, n, f, d, output=mode, exchange=exch)
        for _ in range(2):
            b = fu.aggregate(X).clone()
        torch.cuda.synchronize()
        same = torch.equal(a.view(torch.int32), b.view(torch.int32))
        bad += 0 if same else 1
        print(f"rank {rank} {rule}: {mode} ({fu.fused_path}) exchange={exch} == replicated/nccl: {same}", flush=True)
# deferred barrier: six calls without a barrier, one sync(), then every output
aggs = {r: ShardedAggregator(r, n, f, d, output="fused") for r in ("average", "median", "trimmed_mean", "krum",
                                                                  "multi_krum", "bulyan")}
refs = {r: ShardedAggregator(r, n, f, d, output="replicated", exchange="nccl").aggregate(X).clone() for r in aggs}
for _ in range(3):
    outs = {r: a.aggregate(X, barrier=False) for r, a in aggs.items()}
    aggs["bulyan"].sync()
    torch.cuda.synchronize()
    for r in aggs:
        same = torch.equal(outs[r].view(torch.int32), refs[r].view(torch.int32))
        bad += 0 if same else 1
print(f"rank {rank} deferred-barrier outputs ok: {bad == 0}", flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(1 if bad else 0)
