"""bench.py's JSON-line contract: the reference arm (the oracle
on host cores) on CPU, our arm on a B200.  Small workload (C1), few steps."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def _check_common(j, steps, warmup):
    assert BASE_KEYS <= set(j), BASE_KEYS - set(j)
    assert j["steps"] == steps and j["warmup"] == warmup and j["n_gpus"] == 1
    assert j["value"] > 0 and j["ms_per_step"] > 0 and j["higher_is_better"] is True
    assert j["unit"] == "GB/s" and j["data"] == "synthetic" and j["vs_baseline"] is None
    assert j["config"]["workload"].startswith("C1-") and j["config"]["n"] == 11
    assert set(j["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}


def test_reference_arm_line():
    j = _run("--impl", "reference", "--workload", "C1", "--steps", "3", "--warmup", "3")
    _check_common(j, 3, 3)
    assert j["impl"] == "reference"
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == j["value"] and cb["sample"]
    assert j["e2e"]["value"] == j["value"] and j["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    j = _run("--workload", "C1", "--steps", "3", "--warmup", "3", "--e2e-steps", "2")
    _check_common(j, 3, 3)
    assert "impl" not in j or j["impl"] != "reference"
    rf = j["roofline"]
    assert rf["bound"] in ("hbm", "tensor", "alu") and rf["peak"] > 0 and rf["achieved"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3 and rf["unit"] == "GB/s"
    assert rf["traffic"] is None            # the committed ncu capture is of C3 only
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = j["e2e"]
    n, d = j["config"]["n"], j["config"]["d"]
    # bytes actually copied: rows may carry a few padding coordinates (16-byte aligned leading dimension)
    assert e["value"] > 0 and n * d * 4 <= e["h2d_bytes_per_step"] < n * (d + 64) * 4
    assert 6 * d * 4 <= e["d2h_bytes_per_step"] < 6 * (d + 64) * 4
    assert j["gpu_launches"] > 0 and set(j["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    v = j["variants"]["bf16"]                # the bf16 variant of the same step
    assert v["value"] > 0 and v["ms_per_step"] > 0 and set(v["per_rule"]) == set(j["per_rule"])


@pytest.mark.gpu
def test_our_arm_line_bf16():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    j = _run("--workload", "C1", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--dtype", "bf16")
    _check_common(j, 3, 3)
    assert j["dtype"] == "bf16" and "bf16" in j["metric"]
    n, d = j["config"]["n"], j["config"]["d"]
    e = j["e2e"]
    assert n * d * 2 <= e["h2d_bytes_per_step"] < n * (d + 64) * 2
    assert j["roofline"]["frac"] > 0


def test_roofline_traffic_from_committed_capture():
    """roofline.traffic of the default C3 line = dram read + write per launch of
    the dominant kernel from the committed ncu --set full capture
    (profiles/traffic.json); it must be within 1 % of the kernel's algorithmic
    bytes (n*d*4 read), i.e. no wasted re-reads.  Other workloads: null."""
    import bench
    import synth
    cfg = synth.CONFIGS["C3"]
    t = bench.traffic_from_profiles("gram_tc_kernel<32>", "C3", 1)
    assert t is not None and abs(t / (cfg.n * cfg.d * 4) - 1) < 0.01
    assert bench.traffic_from_profiles("gram_tc_kernel<32>", "C1", 1) is None
    assert bench.traffic_from_profiles("gram_tc_kernel<32>", "C3", 2) is None
