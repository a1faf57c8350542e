"""Boundary tests that need no GPU: libgar.so loads, exports every entry point
include/gar.h declares, and its host-side argument checks return the
documented status codes before any CUDA call (include/gar.h)."""
import ctypes
import filecmp
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gl():
    from paper_2010_05888_b200 import _lib
    return _lib


def test_library_exports_every_declared_symbol(gl):
    declared = gl.header_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(gl.lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", gl.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_kernels_are_sm100a_native(gl):
    """The shared object carries sm_100a SASS (no PTX-JIT / other-arch path)."""
    out = subprocess.run(["cuobjdump", "--list-elf", gl.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", gl.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass or "UTMALDG" in sass          # TMA bulk copies in the coordinate kernel


def test_status_strings(gl):
    for code, name in gl.STATUS.items():
        assert gl.gar_status_string(code) == name


@pytest.mark.parametrize("rule,n,f,m,expect", [
    ("median", 5, 2, 0, 5 * 0), ("median", 4, 2, 0, 0),
    ("krum", 7, 2, 0, 1), ("krum", 6, 2, 0, 0),
    ("multi_krum", 10, 2, 0, 6), ("multi_krum", 10, 2, 3, 3), ("multi_krum", 10, 2, 7, 0),
    ("bulyan", 11, 2, 0, 7), ("bulyan", 10, 2, 0, 0), ("bulyan", 31, 7, 0, 17),
])
def test_num_selected(gl, rule, n, f, m, expect):
    assert gl.gar_num_selected(rule, n, f, m) == expect


def test_workspace_bytes(gl):
    assert gl.gar_workspace_bytes("median", 31, 7, 10**6) == 0
    w = gl.gar_workspace_bytes("bulyan", 31, 7, 10**6)
    assert w >= 31 * 31 * 8
    assert gl.gar_workspace_bytes("bulyan", 30, 7, 10**6) == 0      # quorum violated
    assert gl.gar_workspace_bytes("krum", 65, 0, 10) == 0           # n > 64


def _call_ex(gl, rule, n, f, m, d, ptrs=None, out=0x10_0000, ws=None, wsb=0):
    ptrs = ptrs if ptrs is not None else [0x20_0000 + 0x1000 * i for i in range(n)]
    arr = (ctypes.c_void_p * max(n, 1))(*ptrs)
    return gl.lib.gar_aggregate_ex(gl.rule_id(rule), arr, n, f, m, d, ctypes.c_void_p(out), None,
                                   ctypes.c_void_p(ws) if ws else None, wsb, None)


@pytest.mark.parametrize("rule,n,f,m,code", [
    ("median", 4, 2, 0, 2), ("trimmed_mean", 6, 3, 0, 2), ("krum", 6, 2, 0, 2),
    ("multi_krum", 9, 2, 0, 0), ("multi_krum", 9, 2, 6, 3), ("multi_krum", 9, 2, -1, 3),
    ("bulyan", 10, 2, 0, 2), ("average", 0, 0, 0, 1), ("average", 65, 0, 0, 1), ("median", 5, -1, 0, 1),
])
def test_argument_checks_precede_cuda(gl, rule, n, f, m, code):
    got = _call_ex(gl, rule, n, f, m, 100, ws=0x30_0000 if rule in ("krum", "multi_krum", "bulyan") else None,
                   wsb=1 << 30)
    if code == 0:
        # valid arguments reach the device-pointer check; without a GPU that is a CUDA error
        assert got in (1, 7)
    else:
        assert got == code


def test_alignment_and_aliasing(gl):
    n = 5
    ptrs = [0x20_0000 + 0x1000 * i for i in range(n)]
    ptrs[3] += 4
    assert _call_ex(gl, "median", n, 1, 0, 100, ptrs=ptrs) == 4        # GAR_ERR_ALIGNMENT
    assert _call_ex(gl, "median", n, 1, 0, 100, out=0x10_0008) == 4
    # out overlapping an input row
    assert _call_ex(gl, "median", n, 1, 0, 100, out=0x20_0000 + 0x1000 * 2 + 16) == 1
    # null row
    ptrs = [0x20_0000 + 0x1000 * i for i in range(n)]
    ptrs[1] = 0
    assert _call_ex(gl, "median", n, 1, 0, 100, ptrs=ptrs) == 1
    # Krum family without workspace
    assert _call_ex(gl, "bulyan", 7, 1, 0, 100) == 6


def test_select_rejects_coordinatewise_rules(gl):
    arr = (ctypes.c_void_p * 5)(*[0x20_0000 + 0x1000 * i for i in range(5)])
    nsel = ctypes.c_int(-1)
    code = gl.lib.gar_select(gl.rule_id("median"), arr, 5, 1, 0, 100, ctypes.c_void_p(0x1000), ctypes.byref(nsel),
                             ctypes.c_void_p(0x1000), 1 << 20, None)
    assert code == 5


@pytest.mark.parametrize("rule,n,f,m,code", [
    ("average", 7, 0, 0, 0), ("average", 7, 3, 0, 0), ("average", 7, 9, 0, 0),     # R15: Average ignores f
    ("average", 7, -1, 0, 1), ("median", 7, 3, 0, 0), ("median", 7, 4, 0, 2),
    ("multi_krum", 9, 2, 6, 3), ("multi_krum", 9, 2, 5, 0), ("bulyan", 11, 2, 0, 0), ("bulyan", 10, 2, 0, 2),
    ("mda", 64, 20, 0, 5), ("mda", 9, 3, 0, 0), ("mda", 9, 5, 0, 2), ("median", 65, 0, 0, 1),
])
def test_check_args(gl, rule, n, f, m, code):
    """gar_check_args: the status every entry point's host-side check returns
    (MDA beyond its C(n, f) budget is GAR_ERR_UNSUPPORTED, not a quorum error)."""
    assert gl.gar_check_args(rule, n, f, m) == code


def test_average_accepts_any_f(gl):
    """Reading R15: Average, the non-robust control, ignores f
    (SPEC S:34 asks f = 0); the argument checks pass for any f >= 0."""
    for f in (0, 1, 7, 40):
        assert _call_ex(gl, "average", 31, f, 0, 100) in (1, 7)      # past the checks: device-pointer / CUDA stage
    from paper_2010_05888_b200 import init
    assert init("average", 31, 7).f == 7


def test_mda_budget_reports_unsupported():
    from paper_2010_05888_b200 import init, GarError
    with pytest.raises(GarError) as e:
        init("mda", 64, 20)
    assert e.value.code == 5


def test_python_binding_validates_before_gpu():
    import torch
    from paper_2010_05888_b200 import init, GarError
    with pytest.raises(GarError):
        init("bulyan", 10, 2)
    with pytest.raises(GarError):
        init("multi_krum", 10, 2, m=7)
    with pytest.raises(ValueError):
        init("geometric_median", 10, 2)
    g = init("median", 5, 2)
    with pytest.raises(ValueError):          # CPU tensors are rejected: no CPU fallback
        g.aggregate([torch.zeros(8) for _ in range(5)])


def test_networks_header_is_reproducible(tmp_path):
    gen = os.path.join(ROOT, "paper_2010_05888_b200", "csrc", "gen_networks.py")
    out = tmp_path / "networks.cuh"
    subprocess.check_call([sys.executable, gen, str(out)])
    assert filecmp.cmp(out, os.path.join(ROOT, "paper_2010_05888_b200", "csrc", "networks.cuh"), shallow=False)


def test_bcast_entry_points_check_their_extra_outputs(gl):
    n = 5
    ptrs = (ctypes.c_void_p * n)(*[0x20_0000 + 0x1000 * i for i in range(n)])
    def agg(extra, n_extra):
        arr = (ctypes.c_void_p * max(len(extra), 1))(*extra)
        return gl.lib.gar_aggregate_bcast(gl.rule_id("median"), ptrs, n, 1, 0, 100, ctypes.c_void_p(0x10_0000),
                                          arr, n_extra, None, None, 0, None)
    assert agg([0x40_0000 + 4], 1) == 4            # misaligned extra destination
    assert agg([0], 1) == 1                        # null extra destination
    assert agg([0x40_0000] * 9, 9) == 1            # more than GAR_MAX_PEERS
    assert agg([0x40_0000], -1) == 1
    assert agg([0x40_0000], 1) in (1, 7)           # valid: reaches the device check (no GPU here)
    arr = (ctypes.c_void_p * 1)(0x40_0000)
    code = gl.lib.gar_combine_bcast(gl.rule_id("median"), ptrs, n, 1, 0, 100, ctypes.c_void_p(0x1000),
                                    ctypes.c_void_p(0x10_0000), arr, 1, None)
    assert code == 5                               # combine is for the Krum family


def test_mcast_entry_points_check_their_destination(gl):
    n = 5
    ptrs = (ctypes.c_void_p * n)(*[0x20_0000 + 0x1000 * i for i in range(n)])

    def agg(mc):
        return gl.lib.gar_aggregate_mcast(gl.rule_id("median"), ptrs, n, 1, 0, 100, ctypes.c_void_p(0x10_0000),
                                          ctypes.c_void_p(mc), None, None, 0, None)
    assert agg(0) == 1                             # null multicast address
    assert agg(0x40_0000 + 8) == 4                 # misaligned
    assert agg(0x40_0000) in (1, 7)                # valid: reaches the device check (no GPU here)
    code = gl.lib.gar_combine_mcast(gl.rule_id("median"), ptrs, n, 1, 0, 100, ctypes.c_void_p(0x1000),
                                    ctypes.c_void_p(0x10_0000), ctypes.c_void_p(0x40_0000), None)
    assert code == 5                               # combine is for the Krum family


def test_gram_exchange_checks_its_peer_arrays(gl):
    n = 5
    ptrs = (ctypes.c_void_p * n)(*[0x20_0000 + 0x1000 * i for i in range(n)])

    def call(slots, flags, rank, world):
        sa = (ctypes.c_void_p * max(len(slots), 1))(*slots)
        fa = (ctypes.c_void_p * max(len(flags), 1))(*flags)
        return gl.lib.gar_gram_exchange(ptrs, n, 100, sa, fa, rank, world, 1, ctypes.c_void_p(0x50_0000), None,
                                        ctypes.c_void_p(0x60_0000), 1 << 30, None)
    ok_s, ok_f = [0x70_0000, 0x71_0000], [0x72_0000, 0x73_0000]
    assert call(ok_s, ok_f, 2, 2) == 1                  # rank outside [0, world)
    assert call(ok_s * 5, ok_f * 5, 0, 10) == 1         # world > 8
    assert call([0x70_0000, 0], ok_f, 0, 2) == 1         # null slot array
    assert call([0x70_0004, 0x71_0000], ok_f, 0, 2) == 4  # misaligned slot array
    assert call(ok_s, ok_f, 1, 2) in (1, 7)             # valid: reaches the device check (no GPU here)


def test_mda_arguments(gl):
    """MDA: quorum n >= 2f+1, n - f selected, enumeration
    budget C(n, f) <= 2^31 (GAR_ERR_UNSUPPORTED above)."""
    assert gl.gar_num_selected("mda", 11, 2, 0) == 9
    assert gl.gar_num_selected("mda", 4, 2, 0) == 0
    assert gl.gar_workspace_bytes("mda", 31, 7, 100) > 0
    assert _call_ex(gl, "mda", 4, 2, 0, 100, ws=0x30_0000, wsb=1 << 30) == 2
    assert _call_ex(gl, "mda", 64, 30, 0, 100, ws=0x30_0000, wsb=1 << 30) == 5
    assert _call_ex(gl, "mda", 31, 7, 0, 100, ws=0x30_0000, wsb=1 << 30) in (1, 7)
