"""compute-sanitizer racecheck / synccheck / memcheck over every libgar
kernel family on small inputs: the mbarrier / TMA /
tcgen05 pipelines and the peer-exchange flag protocol must report no
shared-memory hazards, no barrier misuse and no out-of-bounds access."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TARGET = os.path.join(ROOT, "tools", "sanitize_target.py")


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    return None


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = _sanitizer()
    if cs is None:
        pytest.skip("compute-sanitizer not found")
    cmd = [cs, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    r = subprocess.run(cmd + [sys.executable, TARGET], cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    if r.returncode == 86 and "closed on this pool" in out:
        # the GPU pool's wrapper refuses compute-sanitizer (it has left GPUs
        # needing a reset); the run is recorded in profiles/r2_sanitizer.md
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, out[-6000:]
    assert "sanitize target ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
