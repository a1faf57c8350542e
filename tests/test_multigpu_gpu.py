"""The d-sharded multi-GPU path on >= 2 real GPUs: a
torchrun job (tools/multigpu_check.py) runs every rule in every output mode
(NCCL all-gather, peer-memory Gram exchange, fused peer stores, NVLS
multicast, sharded) and compares the replicated aggregate of the whole vectors
bit for bit -- and the selections exactly -- with the ORACLE, fp32 and bf16
rows.  Skips below 2 GPUs (the 1-GPU box runs the fake-rank version,
tests/test_exchange_gpu.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_sharded_paths_against_oracle():
    import torch
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = min(4, torch.cuda.device_count())
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tools", "multigpu_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-6000:]
    assert "multigpu check: ok" in out, out[-3000:]
