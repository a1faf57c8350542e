import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
rank = int(os.environ["RANK"]); torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
buf = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
h = symm_mem.rendezvous(buf, dist.group.WORLD)
from torch._C._distributed_c10d import _SymmetricMemory
print(rank, "has_multicast_support", _SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA, rank),
      "multicast_ptr", h.multicast_ptr, flush=True)
dist.destroy_process_group()
