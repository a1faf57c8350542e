"""ctypes binding of libgar.so (include/gar.h) — argument marshalling only.

Every function here has the name of the C entry point it wraps and takes
torch tensors (device memory) where the C call takes device pointers.  No
step of the method runs in Python; there is no CPU fallback: the library is
loaded on the first C call, and if libgar.so is missing or was built without
the kernels that call raises ImportError.  (Loading lazily lets the package --
and its builder -- be imported on a clean checkout before anything is built.)
"""
from __future__ import annotations

import ctypes
import os
import re

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# GAR_LIB_VARIANT: tools/ experiment builds (libgar_<variant>.so); never set by the product
LIB_PATH = os.path.join(_HERE, "libgar.so" if not os.environ.get("GAR_LIB_VARIANT") else
                        "libgar_" + os.environ["GAR_LIB_VARIANT"] + ".so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "gar.h")

RULES = {"average": 0, "median": 1, "trimmed_mean": 2, "krum": 3, "multi_krum": 4, "bulyan": 5, "mda": 6,
         "mean_around_median": 7}
STATUS = {0: "GAR_OK", 1: "GAR_ERR_INVALID_ARGUMENT", 2: "GAR_ERR_QUORUM", 3: "GAR_ERR_INVALID_M",
          4: "GAR_ERR_ALIGNMENT", 5: "GAR_ERR_UNSUPPORTED", 6: "GAR_ERR_WORKSPACE", 7: "GAR_ERR_CUDA"}
MAX_N = 64
# gar_dtype (include/gar.h): element type of the gradient rows
DTYPES = {torch.float32: 0, torch.bfloat16: 1}


class GarError(RuntimeError):
    def __init__(self, code: int, what: str, detail: str = ""):
        super().__init__(f"{what}: {STATUS.get(code, code)}" + (f" [{detail}]" if detail else ""))
        self.code = code
        self.status = STATUS.get(code, str(code))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libgar.so not built ({LIB_PATH}); run `python -m paper_2010_05888_b200.build` "
                          "(nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
    PP = ctypes.POINTER(ctypes.c_void_p)
    IP = ctypes.POINTER(ctypes.c_int)
    sigs = {
        "gar_status_string": ([I], ctypes.c_char_p),
        "gar_last_error": ([], ctypes.c_char_p),
        "gar_workspace_bytes": ([I, I, I, I64], SZ),
        "gar_num_selected": ([I, I, I, I], I),
        "gar_check_args": ([I, I, I, I], I),
        "gar_aggregate": ([I, PP, I, I, I64, P, P], I),
        "gar_aggregate_ex": ([I, PP, I, I, I, I64, P, P, P, SZ, P], I),
        "gar_select": ([I, PP, I, I, I, I64, P, IP, P, SZ, P], I),
        "gar_distances": ([PP, I, I64, P, P, SZ, P], I),
        "gar_gram_partial": ([PP, I, I64, P, P, SZ, P], I),
        "gar_select_from_gram": ([I, P, I, I, I, P, IP, P, SZ, P], I),
        "gar_combine": ([I, PP, I, I, I, I64, P, P, P], I),
        "gar_aggregate_bcast": ([I, PP, I, I, I, I64, P, PP, I, P, P, SZ, P], I),
        "gar_combine_bcast": ([I, PP, I, I, I, I64, P, P, PP, I, P], I),
        "gar_aggregate_mcast": ([I, PP, I, I, I, I64, P, P, P, P, SZ, P], I),
        "gar_combine_mcast": ([I, PP, I, I, I, I64, P, P, P, P], I),
        "gar_trimmed_membership": ([PP, I, I, I64, P, P], I),
        "gar_nonfinite_rows": ([PP, I, I64, P, P], I),
        "gar_gram_exchange": ([PP, I, I64, PP, PP, I, I, ctypes.c_uint32, P, PP, P, SZ, P], I),
        "gar_aggregate_sgd": ([I, PP, I, I, I, I64, P, ctypes.c_float, P, P, SZ, P], I),
        "gar_combine_sgd": ([I, PP, I, I, I, I64, P, P, ctypes.c_float, P], I),
        "gar_aggregate_dt": ([I, I, PP, I, I, I, I64, P, P, P, SZ, P], I),
        "gar_select_dt": ([I, I, PP, I, I, I, I64, P, IP, P, SZ, P], I),
        "gar_distances_dt": ([I, PP, I, I64, P, P, SZ, P], I),
        "gar_gram_partial_dt": ([I, PP, I, I64, P, P, SZ, P], I),
        "gar_combine_dt": ([I, I, PP, I, I, I, I64, P, P, P], I),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


class _LazyLib:
    """libgar.so, loaded (and its signatures declared) on first attribute access."""

    _cdll = None

    def __getattr__(self, name):
        if _LazyLib._cdll is None:
            _LazyLib._cdll = _load()
        return getattr(_LazyLib._cdll, name)

    @staticmethod
    def loaded() -> bool:
        return _LazyLib._cdll is not None


lib = _LazyLib()


def header_functions() -> list[str]:
    """Entry points declared in include/gar.h (for the export test)."""
    with open(HEADER) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"^(?:gar_status|size_t|int|const char\*)\s+(gar_\w+)\s*\(", src, re.M)))


# ------------------------------------------------------------------ marshalling
def rule_id(rule) -> int:
    if isinstance(rule, str):
        if rule not in RULES:
            raise ValueError(f"unknown GAR {rule!r}; expected one of {sorted(RULES)}")
        return RULES[rule]
    return int(rule)


_PTR_CACHE: dict = {}


class DevicePtrRows:
    """n gradient rows given by raw device addresses (ints), e.g. rows read in
    place from other GPUs' memory over NVLink (dist.WorkerShards).  The
    addresses must be 16-byte aligned and hold >= d fp32 values."""

    def __init__(self, ptrs, device):
        self.ptrs = [int(p) for p in ptrs]
        self.device = torch.device(device)
        self._arr = (ctypes.c_void_p * max(len(self.ptrs), 1))(*self.ptrs)

    def __len__(self):
        return len(self.ptrs)


def row_pointers(grads, d: int | None = None):
    """(ctypes void* array, n, d, device) from a list of 1-D fp32 CUDA tensors
    or a 2-D [n, ld] fp32 CUDA tensor with unit column stride.  For a matrix
    the row pointers are base + i * row_stride (no per-row tensor views), and
    the ctypes array is cached per (base, n, stride)."""
    return row_pointers_dt(grads, d, (torch.float32,))[:4]


def row_pointers_dt(grads, d: int | None = None, dtypes=(torch.float32, torch.bfloat16)):
    """row_pointers for rows of any dtype in `dtypes`; returns (array, n, d,
    device, gar_dtype code).  Raw DevicePtrRows are fp32 (code 0)."""
    if isinstance(grads, DevicePtrRows):
        n = len(grads)
        if not 1 <= n <= MAX_N:
            raise ValueError(f"n = {n} outside [1, {MAX_N}]")
        if d is None:
            raise ValueError("d is required with raw row addresses")
        return grads._arr, n, d, grads.device, 0
    if isinstance(grads, torch.Tensor):
        if grads.dim() != 2:
            raise ValueError("a gradient matrix must be 2-D [n, ld]")
        if grads.dtype not in dtypes:
            raise TypeError(f"gradients must be {' or '.join(str(t) for t in dtypes)}, not {grads.dtype}")
        if grads.device.type != "cuda":
            raise ValueError("gradients must live on a CUDA device (no CPU fallback)")
        n, ld = grads.shape
        if not 1 <= n <= MAX_N:
            raise ValueError(f"n = {n} outside [1, {MAX_N}]")
        if ld > 1 and grads.stride(1) != 1:
            raise ValueError("gradient rows must be contiguous")
        if d is None:
            d = ld
        elif d > ld:
            raise ValueError("a gradient is shorter than d")
        base, rs = grads.data_ptr(), grads.stride(0) * grads.element_size()
        key = (base, n, rs)
        arr = _PTR_CACHE.get(key)
        if arr is None:
            if len(_PTR_CACHE) > 256:
                _PTR_CACHE.clear()
            arr = (ctypes.c_void_p * n)(*[base + i * rs for i in range(n)])
            _PTR_CACHE[key] = arr
        return arr, n, d, grads.device, DTYPES[grads.dtype]
    rows = list(grads)
    n = len(rows)
    if not 1 <= n <= MAX_N:
        raise ValueError(f"n = {n} outside [1, {MAX_N}]")
    dev = rows[0].device
    dt = rows[0].dtype
    for r in rows:
        if r.dtype not in dtypes or r.dtype != dt:
            raise TypeError(f"gradients must all be {' or '.join(str(t) for t in dtypes)} (one dtype), "
                            f"not {r.dtype}")
        if r.device != dev or r.device.type != "cuda":
            raise ValueError("gradients must all live on the same CUDA device (no CPU fallback)")
        if r.dim() != 1 or (r.numel() > 1 and r.stride(0) != 1):
            raise ValueError("each gradient must be a contiguous 1-D view")
    if d is None:
        d = min(r.numel() for r in rows)
    elif any(r.numel() < d for r in rows):
        raise ValueError("a gradient is shorter than d")
    arr = (ctypes.c_void_p * n)(*[r.data_ptr() for r in rows])
    return arr, n, d, dev, DTYPES[dt]


def stream_handle(device, stream=None):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _idx(indices, rule, n, f, m, dev, optional):
    """Selected-index buffer: int32 on `dev`, room for gar_num_selected."""
    return _buf(indices, torch.int32, max(1, gar_num_selected(rule, n, f, m)), dev, "indices", optional)


def _buf(t, dtype, numel: int, dev, what: str, optional: bool = False):
    """Pointer to a caller buffer after the checks the C ABI cannot make:
    a contiguous CUDA tensor of `dtype` on the gradients' device holding at
    least `numel` elements (None allowed when optional)."""
    if t is None:
        if optional:
            return ctypes.c_void_p(0)
        raise ValueError(f"{what} is required")
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor")
    if t.device.type != "cuda" or (dev is not None and t.device != dev):
        raise ValueError(f"{what} must live on the gradients' CUDA device ({dev}), not {t.device}")
    if t.dtype not in ((dtype,) if not isinstance(dtype, tuple) else dtype):
        raise TypeError(f"{what} must be {dtype}, not {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if t.numel() < numel:
        raise ValueError(f"{what} holds {t.numel()} elements, needs {numel}")
    return ctypes.c_void_p(t.data_ptr())


def check(code: int, what: str):
    if code != 0:
        detail = lib.gar_last_error().decode() if code == 7 else ""
        raise GarError(code, what, detail)


# ------------------------------------------------------------------ same names as the C ABI
def gar_status_string(code: int) -> str:
    return lib.gar_status_string(code).decode()


def gar_last_error() -> str:
    return lib.gar_last_error().decode()


def gar_workspace_bytes(rule, n: int, f: int, d: int) -> int:
    return int(lib.gar_workspace_bytes(rule_id(rule), n, f, d))


def gar_check_args(rule, n: int, f: int, m: int = 0) -> int:
    """The C library's argument status for (rule, n, f, m) (0 = GAR_OK)."""
    return int(lib.gar_check_args(rule_id(rule), n, f, m))


def gar_num_selected(rule, n: int, f: int, m: int = 0) -> int:
    return int(lib.gar_num_selected(rule_id(rule), n, f, m))


def _wsb(workspace) -> int:
    return 0 if workspace is None else workspace.numel() * workspace.element_size()


def _f32(t, d, dev, what="out"):
    return _buf(t, torch.float32, d, dev, what)


def gar_aggregate(rule, grads, f: int, out: torch.Tensor, d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    check(lib.gar_aggregate(rule_id(rule), arr, n, f, d, _f32(out, d, dev), stream_handle(dev, stream)),
          "gar_aggregate")
    return out


def gar_aggregate_ex(rule, grads, f: int, m: int, out: torch.Tensor, indices=None, workspace=None,
                     d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    o, ix = _f32(out, d, dev), _idx(indices, rule, n, f, m, dev, True)
    check(lib.gar_aggregate_ex(rule_id(rule), arr, n, f, m, d, o, ix, _ptr(workspace), _wsb(workspace),
                               stream_handle(dev, stream)), "gar_aggregate_ex")
    return out


def gar_select(rule, grads, f: int, m: int, indices: torch.Tensor, workspace: torch.Tensor,
               d: int | None = None, stream=None) -> int:
    arr, n, d, dev = row_pointers(grads, d)
    nsel = ctypes.c_int(0)
    ix = _idx(indices, rule, n, f, m, dev, False)
    check(lib.gar_select(rule_id(rule), arr, n, f, m, d, ix, ctypes.byref(nsel), _ptr(workspace), _wsb(workspace),
                         stream_handle(dev, stream)), "gar_select")
    return nsel.value


def gar_distances(grads, D: torch.Tensor, workspace: torch.Tensor, d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    dp = _buf(D, torch.float64, n * n, dev, "D")
    check(lib.gar_distances(arr, n, d, dp, _ptr(workspace), _wsb(workspace), stream_handle(dev, stream)),
          "gar_distances")
    return D


def gar_gram_partial(grads, gram: torch.Tensor, workspace: torch.Tensor, d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    g = _buf(gram, torch.float64, n * n, dev, "gram")
    check(lib.gar_gram_partial(arr, n, d, g, _ptr(workspace), _wsb(workspace), stream_handle(dev, stream)),
          "gar_gram_partial")
    return gram


def gar_select_from_gram(rule, gram: torch.Tensor, n: int, f: int, m: int, indices: torch.Tensor,
                         stream=None, workspace: torch.Tensor | None = None) -> int:
    """workspace: required for MDA (gar_workspace_bytes), unused otherwise."""
    nsel = ctypes.c_int(0)
    dev = gram.device
    g, ix = _buf(gram, torch.float64, n * n, dev, "gram"), _idx(indices, rule, n, f, m, dev, False)
    check(lib.gar_select_from_gram(rule_id(rule), g, n, f, m, ix, ctypes.byref(nsel), _ptr(workspace),
                                   _wsb(workspace), stream_handle(dev, stream)), "gar_select_from_gram")
    return nsel.value


def gar_combine(rule, grads, f: int, m: int, indices: torch.Tensor, out: torch.Tensor, d: int | None = None,
                stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    ix, o = _idx(indices, rule, n, f, m, dev, False), _f32(out, d, dev)
    check(lib.gar_combine(rule_id(rule), arr, n, f, m, d, ix, o, stream_handle(dev, stream)), "gar_combine")
    return out


def _ptr_array(addrs):
    addrs = list(addrs)
    return (ctypes.c_void_p * max(len(addrs), 1))(*addrs), len(addrs)


def gar_aggregate_bcast(rule, grads, f: int, m: int, out: torch.Tensor, extra_ptrs, indices=None, workspace=None,
                        d: int | None = None, stream=None):
    """gar_aggregate_ex + the result also stored at each address of extra_ptrs
    (ints: peer-mapped buffers, e.g. torch symmetric memory)."""
    arr, n, d, dev = row_pointers(grads, d)
    ex, ne = _ptr_array(extra_ptrs)
    o, ix = _f32(out, d, dev), _idx(indices, rule, n, f, m, dev, True)
    check(lib.gar_aggregate_bcast(rule_id(rule), arr, n, f, m, d, o, ex, ne, ix, _ptr(workspace), _wsb(workspace),
                                  stream_handle(dev, stream)), "gar_aggregate_bcast")
    return out


def gar_combine_bcast(rule, grads, f: int, m: int, indices: torch.Tensor, out: torch.Tensor, extra_ptrs,
                      d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    ex, ne = _ptr_array(extra_ptrs)
    ix, o = _idx(indices, rule, n, f, m, dev, False), _f32(out, d, dev)
    check(lib.gar_combine_bcast(rule_id(rule), arr, n, f, m, d, ix, o, ex, ne, stream_handle(dev, stream)),
          "gar_combine_bcast")
    return out


def gar_aggregate_mcast(rule, grads, f: int, m: int, out: torch.Tensor, out_mc: int, indices=None, workspace=None,
                        d: int | None = None, stream=None):
    """gar_aggregate_ex with the result stored through the multicast address
    out_mc (an int) that maps `out` on every member GPU."""
    arr, n, d, dev = row_pointers(grads, d)
    o, ix = _f32(out, d, dev), _idx(indices, rule, n, f, m, dev, True)
    check(lib.gar_aggregate_mcast(rule_id(rule), arr, n, f, m, d, o, ctypes.c_void_p(out_mc), ix, _ptr(workspace),
                                  _wsb(workspace), stream_handle(dev, stream)), "gar_aggregate_mcast")
    return out


def gar_combine_mcast(rule, grads, f: int, m: int, indices: torch.Tensor, out: torch.Tensor, out_mc: int,
                      d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    ix, o = _idx(indices, rule, n, f, m, dev, False), _f32(out, d, dev)
    check(lib.gar_combine_mcast(rule_id(rule), arr, n, f, m, d, ix, o, ctypes.c_void_p(out_mc),
                                stream_handle(dev, stream)), "gar_combine_mcast")
    return out


def gar_trimmed_membership(grads, f: int, mask: torch.Tensor, d: int | None = None, stream=None):
    """mask: device int64[d] (uint64 bit patterns): bit i set iff input i is kept
    by the trimmed mean at that coordinate."""
    arr, n, d, dev = row_pointers(grads, d)
    mk = _buf(mask, (torch.int64, torch.uint64), d, dev, "mask")
    check(lib.gar_trimmed_membership(arr, n, f, d, mk, stream_handle(dev, stream)), "gar_trimmed_membership")
    return mask


def gar_gram_exchange(grads, gram: torch.Tensor, workspace: torch.Tensor, peer_slots, peer_flags, rank: int,
                      world: int, epoch: int, d: int | None = None, stream=None, stage: torch.Tensor | None = None):
    """Whole-vector Gram matrix of d-sharded rows, exchanged over peer memory
    (ints peer_slots / peer_flags: every rank's slot / flag arrays).  stage:
    optional [n, >= d] fp32 matrix that receives a local copy of the rows."""
    arr, n, d, dev = row_pointers(grads, d)
    sl, _ = _ptr_array(peer_slots)
    fl, _ = _ptr_array(peer_flags)
    g = _buf(gram, torch.float64, n * n, dev, "gram")
    st = None
    if stage is not None:
        if stage.dim() != 2 or stage.shape[0] != n or stage.shape[1] < d or stage.stride(1) != 1:
            raise ValueError("stage must be an [n, >= d] row-major fp32 matrix")
        st, _, _, _ = row_pointers(stage, d)
    check(lib.gar_gram_exchange(arr, n, d, sl, fl, rank, world, epoch, g, st, _ptr(workspace), _wsb(workspace),
                                stream_handle(dev, stream)), "gar_gram_exchange")
    return gram


def gar_aggregate_sgd(rule, grads, f: int, m: int, params: torch.Tensor, lr: float, indices=None, workspace=None,
                      d: int | None = None, stream=None):
    """params <- params - lr * GAR(grads), fused into the producing kernel."""
    arr, n, d, dev = row_pointers(grads, d)
    pp, ix = _f32(params, d, dev, "params"), _idx(indices, rule, n, f, m, dev, True)
    check(lib.gar_aggregate_sgd(rule_id(rule), arr, n, f, m, d, pp, float(lr), ix, _ptr(workspace), _wsb(workspace),
                                stream_handle(dev, stream)), "gar_aggregate_sgd")
    return params


def gar_combine_sgd(rule, grads, f: int, m: int, indices: torch.Tensor, params: torch.Tensor, lr: float,
                    d: int | None = None, stream=None):
    arr, n, d, dev = row_pointers(grads, d)
    ix, pp = _idx(indices, rule, n, f, m, dev, False), _f32(params, d, dev, "params")
    check(lib.gar_combine_sgd(rule_id(rule), arr, n, f, m, d, ix, pp, float(lr), stream_handle(dev, stream)),
          "gar_combine_sgd")
    return params


def gar_nonfinite_rows(grads, mask: torch.Tensor, d: int | None = None, stream=None):
    """mask: device int64[>= 1]; mask[0] bit i set iff row i holds a NaN/inf."""
    arr, n, d, dev = row_pointers(grads, d)
    mk = _buf(mask, (torch.int64, torch.uint64), 1, dev, "mask")
    check(lib.gar_nonfinite_rows(arr, n, d, mk, stream_handle(dev, stream)), "gar_nonfinite_rows")
    return mask


# ------------------------------------------------------------------ bf16 rows (gar.h "_dt" entry points)
def gar_aggregate_dt(rule, grads, f: int, m: int, out: torch.Tensor, indices=None, workspace=None,
                     d: int | None = None, stream=None):
    """gar_aggregate_ex for fp32 or bf16 rows (dtype from the tensors); out fp32."""
    arr, n, d, dev, dt = row_pointers_dt(grads, d)
    o, ix = _f32(out, d, dev), _idx(indices, rule, n, f, m, dev, True)
    check(lib.gar_aggregate_dt(rule_id(rule), dt, arr, n, f, m, d, o, ix, _ptr(workspace), _wsb(workspace),
                               stream_handle(dev, stream)), "gar_aggregate_dt")
    return out


def gar_select_dt(rule, grads, f: int, m: int, indices: torch.Tensor, workspace: torch.Tensor,
                  d: int | None = None, stream=None) -> int:
    arr, n, d, dev, dt = row_pointers_dt(grads, d)
    nsel = ctypes.c_int(0)
    ix = _idx(indices, rule, n, f, m, dev, False)
    check(lib.gar_select_dt(rule_id(rule), dt, arr, n, f, m, d, ix, ctypes.byref(nsel), _ptr(workspace),
                            _wsb(workspace), stream_handle(dev, stream)), "gar_select_dt")
    return nsel.value


def gar_distances_dt(grads, D: torch.Tensor, workspace: torch.Tensor, d: int | None = None, stream=None):
    arr, n, d, dev, dt = row_pointers_dt(grads, d)
    dp = _buf(D, torch.float64, n * n, dev, "D")
    check(lib.gar_distances_dt(dt, arr, n, d, dp, _ptr(workspace), _wsb(workspace), stream_handle(dev, stream)),
          "gar_distances_dt")
    return D


def gar_gram_partial_dt(grads, gram: torch.Tensor, workspace: torch.Tensor, d: int | None = None, stream=None):
    arr, n, d, dev, dt = row_pointers_dt(grads, d)
    g = _buf(gram, torch.float64, n * n, dev, "gram")
    check(lib.gar_gram_partial_dt(dt, arr, n, d, g, _ptr(workspace), _wsb(workspace), stream_handle(dev, stream)),
          "gar_gram_partial_dt")
    return gram


def gar_combine_dt(rule, grads, f: int, m: int, indices: torch.Tensor, out: torch.Tensor, d: int | None = None,
                   stream=None):
    arr, n, d, dev, dt = row_pointers_dt(grads, d)
    ix, o = _idx(indices, rule, n, f, m, dev, False), _f32(out, d, dev)
    check(lib.gar_combine_dt(rule_id(rule), dt, arr, n, f, m, d, ix, o, stream_handle(dev, stream)),
          "gar_combine_dt")
    return out
