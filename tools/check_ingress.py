"""torchrun: d-sharded GARs reading the worker-major gradients in place over
NVLink (dist.WorkerShards) vs the pre-sharded layout: outputs
bit-identical on every rank; per-rule device time of both (max over ranks)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import synth
from paper_2010_05888_b200.dist import ShardedAggregator, WorkerShards, shard_bounds

local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synth.CONFIGS[wl]
n, f, d = cfg.n, cfg.f, cfg.d
full = synth.make_gradients(n, f, d, seed=synth.BASE_SEED + 77, device=dev)     # same on every rank
lo, hi = shard_bounds(d, rank, world)
X_local = full[:, lo:hi].contiguous()
ws = WorkerShards(n, d, device=dev)
rows = ws.local_rows()
for j, w in enumerate(ws.local_workers):
    rows[j, :d].copy_(full[w, :d])
del full
torch.cuda.synchronize()
ws.ready()
peer_rows = ws.slice_rows(lo)
bad, res = 0, {}
for rule in ("average", "median", "trimmed_mean", "krum", "multi_krum", "bulyan"):
    a = ShardedAggregator(rule, n, f, d, output="sharded")
    b = ShardedAggregator(rule, n, f, d, output="sharded")
    ra = a.aggregate(X_local).clone()
    rb = b.aggregate(peer_rows).clone()
    torch.cuda.synchronize()
    same = torch.equal(ra.view(torch.int32), rb.view(torch.int32))
    bad += 0 if same else 1

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(); dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record(); torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / reps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return round(float(t), 4)
    res[rule] = {"same": same, "presharded_ms": timed(lambda: a.aggregate(X_local)),
                 "peer_ingress_ms": timed(lambda: b.aggregate(peer_rows))}
if rank == 0:
    print(json.dumps({"workload": wl, "world": world, "per_rule": res}), flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(1 if bad else 0)
