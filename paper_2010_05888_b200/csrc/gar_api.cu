// gar_api.cu — the C-ABI of libgar (include/gar.h): argument checks, workspace
// carving and kernel sequencing.  No arithmetic of the method happens on the
// host; every step runs in the kernels of coord_select*.cu, gram_*.cu and
// select.cu.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/gar.h"
#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "gram.h"

namespace {

using gar::CoordLaunch;

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// The selection rules: Gram matrix -> selected inputs -> combine.
bool is_krum_family(gar_rule r) {
  return r == GAR_KRUM || r == GAR_MULTI_KRUM || r == GAR_BULYAN || r == GAR_MDA;
}

bool valid_rule(int r) { return r >= GAR_AVERAGE && r <= GAR_MEAN_AROUND_MEDIAN; }

// Effective m for (rule, n, f, m): Krum 1, Multi-Krum m (0 -> n-f-2), MDA n-f.
int effective_m(gar_rule rule, int n, int f, int m) {
  if (rule == GAR_KRUM) return 1;
  if (rule == GAR_MULTI_KRUM) return m == 0 ? n - f - 2 : m;
  if (rule == GAR_MDA) return n - f;
  return 0;
}

// MDA enumerates the C(n, f) excluded sets: bounded (~2e9 subsets, seconds).
constexpr uint64_t kMdaMaxSubsets = 1ull << 31;
bool mda_within_budget(int n, int f) {
  uint64_t c = 1;
  for (int i = 1; i <= f; ++i) {
    c = c * uint64_t(n - f + i) / uint64_t(i);
    if (c > kMdaMaxSubsets) return false;
  }
  return true;
}

// Pure argument checks (no CUDA calls): rule, sizes, quorum (PAPER.md l.208,
// l.210-212, l.225), m.
gar_status check_rule_args(gar_rule rule, int n, int f, int m) {
  if (!valid_rule(rule) || n < 1 || n > GAR_MAX_N || f < 0) return GAR_ERR_INVALID_ARGUMENT;
  switch (rule) {
    case GAR_AVERAGE: return GAR_OK;
    case GAR_MEDIAN:
    case GAR_TRIMMED_MEAN:
    case GAR_MEAN_AROUND_MEDIAN: return n >= 2 * f + 1 ? GAR_OK : GAR_ERR_QUORUM;
    case GAR_KRUM:
    case GAR_MULTI_KRUM: {
      if (n < 2 * f + 3) return GAR_ERR_QUORUM;
      const int me = effective_m(rule, n, f, m);
      if (m < 0 || me < 1 || me > n - f - 2) return GAR_ERR_INVALID_M;
      return GAR_OK;
    }
    case GAR_BULYAN: return n >= 4 * f + 3 ? GAR_OK : GAR_ERR_QUORUM;
    case GAR_MDA:
      if (n < 2 * f + 1) return GAR_ERR_QUORUM;
      return mda_within_budget(n, f) ? GAR_OK : GAR_ERR_UNSUPPORTED;
  }
  return GAR_ERR_INVALID_ARGUMENT;
}

gar_status check_rows(const float* const* grads, int n, int64_t d) {
  if (!grads || d < 0) return GAR_ERR_INVALID_ARGUMENT;
  for (int i = 0; i < n; ++i) {
    if (!grads[i]) return GAR_ERR_INVALID_ARGUMENT;
    if (reinterpret_cast<uintptr_t>(grads[i]) & 15u) return GAR_ERR_ALIGNMENT;
  }
  return GAR_OK;
}

bool valid_dtype(int t) { return t == GAR_F32 || t == GAR_BF16; }
uintptr_t elem_bytes(gar_dtype t) { return t == GAR_BF16 ? 2u : 4u; }

gar_status check_out(const float* const* grads, int n, int64_t d, const float* out, gar_dtype dt = GAR_F32) {
  if (!out) return GAR_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(out) & 15u) return GAR_ERR_ALIGNMENT;
  const uintptr_t o0 = reinterpret_cast<uintptr_t>(out), o1 = o0 + uintptr_t(d) * 4u;
  for (int i = 0; i < n; ++i) {
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(grads[i]), g1 = g0 + uintptr_t(d) * elem_bytes(dt);
    if (d > 0 && o0 < g1 && g0 < o1) return GAR_ERR_INVALID_ARGUMENT;
  }
  return GAR_OK;
}

thread_local char g_last_error[256] = "";

inline gar_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return GAR_OK;
  std::snprintf(g_last_error, sizeof(g_last_error), "%s (%d)", cudaGetErrorString(e), static_cast<int>(e));
  cudaGetLastError();   // clear non-sticky errors so the next call starts clean
  return GAR_ERR_CUDA;
}

// Device-pointer check (no CPU fallback: host memory is rejected).
gar_status check_device_ptr(const void* p) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    if (e == cudaErrorInvalidValue) {
      cudaGetLastError();
      return GAR_ERR_INVALID_ARGUMENT;
    }
    return cuda_status(e);
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return GAR_ERR_INVALID_ARGUMENT;
  return GAR_OK;
}

// Pointer-table validation costs one cudaPointerGetAttributes per row; a
// per-thread cache of recently validated (device, table) pairs lets repeated
// calls on the same gradient buffers (the normal training-loop case) skip it.
struct ValidatedSet {
  int device = -1;
  int n = 0;
  const float* p[GAR_MAX_N];
};
thread_local ValidatedSet g_validated[4];
thread_local int g_validated_next = 0;

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  return dev;
}

gar_status check_device_rows(const float* const* grads, int n, const void* out) {
  const int dev = current_device();
  bool cached = false;
  for (const ValidatedSet& v : g_validated) {
    if (v.device == dev && v.n == n && std::memcmp(v.p, grads, sizeof(const float*) * n) == 0) {
      cached = true;
      break;
    }
  }
  if (!cached) {
    for (int i = 0; i < n; ++i) {
      gar_status s = check_device_ptr(grads[i]);
      if (s != GAR_OK) return s;
    }
    ValidatedSet& v = g_validated[g_validated_next];
    g_validated_next = (g_validated_next + 1) % 4;
    v.device = dev;
    v.n = n;
    std::memcpy(v.p, grads, sizeof(const float*) * n);
  }
  return out ? check_device_ptr(out) : GAR_OK;
}

int num_sms() {
  static int cache[64] = {0};
  const int dev = current_device();
  if (dev < 0) return 148;
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  if (dev < 64) cache[dev] = sms;
  return sms;
}

// Workspace layout (Krum family): [partials | G | idx], 256-byte aligned parts.
struct Workspace {
  double* partials;
  double* G;
  int32_t* idx;
  double* D;       // MDA: the distance matrix
  void* mda;       // MDA: enumeration scratch
};

size_t ws_bytes_for(int n) {
  size_t b = align_up(sizeof(double) * gar::kGramMaxParts * n * n, 256);
  b += align_up(sizeof(double) * n * n, 256);
  b += align_up(sizeof(int32_t) * GAR_MAX_N, 256);
  b += align_up(sizeof(double) * n * n, 256);
  b += align_up(gar::mda_workspace_bytes(n), 256);
  return b;
}

Workspace carve(void* ws, int n) {
  unsigned char* p = static_cast<unsigned char*>(ws);
  Workspace w;
  w.partials = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * gar::kGramMaxParts * n * n, 256);
  w.G = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * n * n, 256);
  w.idx = reinterpret_cast<int32_t*>(p);
  p += align_up(sizeof(int32_t) * GAR_MAX_N, 256);
  w.D = reinterpret_cast<double*>(p);
  p += align_up(sizeof(double) * n * n, 256);
  w.mda = p;
  return w;
}

gar_status run_gram(const float* const* grads, int n, int64_t d, const Workspace& w, cudaStream_t st,
                    gar_dtype dt = GAR_F32) {
  int parts = 0;
  gar_status s =
      cuda_status(gar::launch_gram_partials(grads, n, d, w.partials, num_sms(), &parts, st, nullptr, dt));
  if (s != GAR_OK) return s;
  return cuda_status(gar::launch_gram_reduce(w.partials, parts, n, w.G, st));
}

gar_status run_select(gar_rule rule, const double* G, int n, int f, int me, int32_t* idx, double* D_out,
                      const Workspace* w, cudaStream_t st) {
  if (rule == GAR_MDA) {
    if (!w) return GAR_ERR_WORKSPACE;
    gar_status s = cuda_status(gar::launch_select(G, n, 0, 0, gar::kSelDistancesOnly, w->idx, w->D, st));
    if (s != GAR_OK) return s;
    return cuda_status(gar::launch_mda_select(w->D, n, f, w->mda, num_sms(), idx, st));
  }
  const int srule = (rule == GAR_BULYAN) ? gar::kSelBulyan : gar::kSelMultiKrum;
  return cuda_status(gar::launch_select(G, n, f, me, srule, idx, D_out, st));
}

gar_status run_combine(gar_rule rule, const float* const* grads, int n, int f, int me, int64_t d,
                       const int32_t* idx, float* out, const gar::OutPtrs& extra, cudaStream_t st,
                       gar_dtype dt = GAR_F32) {
  CoordLaunch L{};
  L.dtype = dt;
  L.rows = grads;
  L.n = n;
  L.idx = idx;
  L.f = f;
  L.d = d;
  L.out = out;
  L.extra = extra;
  L.num_sms = num_sms();
  if (rule == GAR_BULYAN) {
    L.R = n - 2 * f;
    return cuda_status(gar::launch_coord_select(gar::kModeBulyan, L, st));
  }
  L.R = me;
  return cuda_status(gar::launch_coord_select(gar::kModeAverage, L, st));
}

// Extra destinations of the broadcast variants: non-null, 16-byte aligned, at
// most GAR_MAX_PEERS; they may be peer-mapped (symmetric) memory, so they are
// not checked with cudaPointerGetAttributes.
gar_status make_extra(float* const* extra_outs, int n_extra, gar::OutPtrs* extra) {
  extra->n = 0;
  if (n_extra < 0 || n_extra > GAR_MAX_PEERS || (n_extra > 0 && !extra_outs)) return GAR_ERR_INVALID_ARGUMENT;
  for (int j = 0; j < n_extra; ++j) {
    if (!extra_outs[j]) return GAR_ERR_INVALID_ARGUMENT;
    if (reinterpret_cast<uintptr_t>(extra_outs[j]) & 15u) return GAR_ERR_ALIGNMENT;
    extra->p[j] = extra_outs[j];
  }
  extra->n = n_extra;
  return GAR_OK;
}

// Multicast destination (NVLS): non-null, 16-byte aligned; a multicast
// virtual address is not checked with cudaPointerGetAttributes.
gar_status make_mc(float* out_mc, gar::OutPtrs* extra) {
  *extra = gar::OutPtrs{};
  if (!out_mc) return GAR_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(out_mc) & 15u) return GAR_ERR_ALIGNMENT;
  extra->mc = out_mc;
  return GAR_OK;
}

gar_status aggregate_impl(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d, float* out,
                          const gar::OutPtrs& extra, int32_t* indices_dev, void* workspace, size_t workspace_bytes,
                          gar_stream_t stream, gar_dtype dt = GAR_F32) {
  if (!valid_dtype(dt)) return GAR_ERR_INVALID_ARGUMENT;
  gar_status s = check_rule_args(rule, n, f, m);
  if (s != GAR_OK) return s;
  if ((s = check_rows(grads, n, d)) != GAR_OK) return s;
  if ((s = check_out(grads, n, d, out, dt)) != GAR_OK) return s;
  const bool krum = is_krum_family(rule);
  if (krum && (!workspace || workspace_bytes < ws_bytes_for(n))) return GAR_ERR_WORKSPACE;
  if ((s = check_device_rows(grads, n, out)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);

  if (!krum) {
    CoordLaunch L{};
    L.dtype = dt;
    L.rows = grads;
    L.n = n;
    L.idx = nullptr;
    L.R = n;
    L.f = f;
    L.d = d;
    L.out = out;
    L.extra = extra;
    L.num_sms = num_sms();
    int mode = gar::kModeAverage;
    if (rule == GAR_MEDIAN) mode = gar::kModeMedian;
    if (rule == GAR_TRIMMED_MEAN) mode = gar::kModeTrimmed;
    // mean around median = Bulyan's coordinate phase over all n inputs (R14)
    if (rule == GAR_MEAN_AROUND_MEDIAN) mode = gar::kModeBulyan;
    return cuda_status(gar::launch_coord_select(mode, L, st));
  }
  const int me = effective_m(rule, n, f, m);
  Workspace w = carve(workspace, n);
  int32_t* idx = indices_dev ? indices_dev : w.idx;
  if ((s = run_gram(grads, n, d, w, st, dt)) != GAR_OK) return s;
  if ((s = run_select(rule, w.G, n, f, me, idx, nullptr, &w, st)) != GAR_OK) return s;
  return run_combine(rule, grads, n, f, me, d, idx, out, extra, st, dt);
}

gar_status combine_impl(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d_local,
                        const int32_t* indices_dev, float* out, const gar::OutPtrs& extra, gar_stream_t stream,
                        gar_dtype dt = GAR_F32) {
  if (!valid_dtype(dt)) return GAR_ERR_INVALID_ARGUMENT;
  gar_status s = check_rule_args(rule, n, f, m);
  if (s != GAR_OK) return s;
  if (!is_krum_family(rule)) return GAR_ERR_UNSUPPORTED;
  if (!indices_dev) return GAR_ERR_INVALID_ARGUMENT;
  if ((s = check_rows(grads, n, d_local)) != GAR_OK) return s;
  if ((s = check_out(grads, n, d_local, out, dt)) != GAR_OK) return s;
  if ((s = check_device_rows(grads, n, out)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return run_combine(rule, grads, n, f, effective_m(rule, n, f, m), d_local, indices_dev, out, extra, st, dt);
}

gar_status select_impl(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                       int32_t* indices_dev, int* n_selected_host, void* workspace, size_t workspace_bytes,
                       gar_stream_t stream, gar_dtype dt) {
  if (!valid_dtype(dt)) return GAR_ERR_INVALID_ARGUMENT;
  gar_status s = check_rule_args(rule, n, f, m);
  if (s != GAR_OK) return s;
  if (!is_krum_family(rule)) return GAR_ERR_UNSUPPORTED;
  if (!indices_dev) return GAR_ERR_INVALID_ARGUMENT;
  if ((s = check_rows(grads, n, d)) != GAR_OK) return s;
  if (!workspace || workspace_bytes < ws_bytes_for(n)) return GAR_ERR_WORKSPACE;
  if ((s = check_device_rows(grads, n, nullptr)) != GAR_OK) return s;
  if ((s = check_device_ptr(indices_dev)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int me = effective_m(rule, n, f, m);
  Workspace w = carve(workspace, n);
  if ((s = run_gram(grads, n, d, w, st, dt)) != GAR_OK) return s;
  if ((s = run_select(rule, w.G, n, f, me, indices_dev, nullptr, &w, st)) != GAR_OK) return s;
  if (n_selected_host) *n_selected_host = gar_num_selected(rule, n, f, m);
  return GAR_OK;
}

gar_status distances_impl(const float* const* grads, int n, int64_t d, double* D_dev, void* workspace,
                          size_t workspace_bytes, gar_stream_t stream, gar_dtype dt) {
  if (!valid_dtype(dt)) return GAR_ERR_INVALID_ARGUMENT;
  if (n < 1 || n > GAR_MAX_N || !D_dev) return GAR_ERR_INVALID_ARGUMENT;
  gar_status s = check_rows(grads, n, d);
  if (s != GAR_OK) return s;
  if (!workspace || workspace_bytes < ws_bytes_for(n)) return GAR_ERR_WORKSPACE;
  if ((s = check_device_rows(grads, n, nullptr)) != GAR_OK) return s;
  if ((s = check_device_ptr(D_dev)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace w = carve(workspace, n);
  if ((s = run_gram(grads, n, d, w, st, dt)) != GAR_OK) return s;
  return cuda_status(gar::launch_select(w.G, n, 0, 0, gar::kSelDistancesOnly, w.idx, D_dev, st));
}

gar_status gram_partial_impl(const float* const* grads, int n, int64_t d_local, double* gram_dev, void* workspace,
                             size_t workspace_bytes, gar_stream_t stream, gar_dtype dt) {
  if (!valid_dtype(dt)) return GAR_ERR_INVALID_ARGUMENT;
  if (n < 1 || n > GAR_MAX_N || !gram_dev) return GAR_ERR_INVALID_ARGUMENT;
  gar_status s = check_rows(grads, n, d_local);
  if (s != GAR_OK) return s;
  if (!workspace || workspace_bytes < ws_bytes_for(n)) return GAR_ERR_WORKSPACE;
  if ((s = check_device_rows(grads, n, nullptr)) != GAR_OK) return s;
  if ((s = check_device_ptr(gram_dev)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace w = carve(workspace, n);
  int parts = 0;
  if ((s = cuda_status(gar::launch_gram_partials(grads, n, d_local, w.partials, num_sms(), &parts, st, nullptr,
                                                 dt))) != GAR_OK)
    return s;
  return cuda_status(gar::launch_gram_reduce(w.partials, parts, n, gram_dev, st));
}

// the bf16 entry points take the rows as untyped pointers
inline const float* const* rows_cast(const void* const* grads) {
  return reinterpret_cast<const float* const*>(grads);
}

}  // namespace

extern "C" {

const char* gar_last_error(void) { return g_last_error; }

const char* gar_status_string(gar_status s) {
  switch (s) {
    case GAR_OK: return "GAR_OK";
    case GAR_ERR_INVALID_ARGUMENT: return "GAR_ERR_INVALID_ARGUMENT";
    case GAR_ERR_QUORUM: return "GAR_ERR_QUORUM";
    case GAR_ERR_INVALID_M: return "GAR_ERR_INVALID_M";
    case GAR_ERR_ALIGNMENT: return "GAR_ERR_ALIGNMENT";
    case GAR_ERR_UNSUPPORTED: return "GAR_ERR_UNSUPPORTED";
    case GAR_ERR_WORKSPACE: return "GAR_ERR_WORKSPACE";
    case GAR_ERR_CUDA: return "GAR_ERR_CUDA";
  }
  return "GAR_ERR_UNKNOWN";
}

size_t gar_workspace_bytes(gar_rule rule, int n, int f, int64_t d) {
  if (check_rule_args(rule, n, f, 0) != GAR_OK || d < 0) return 0;
  if (!is_krum_family(rule)) return 0;
  return ws_bytes_for(n);
}

gar_status gar_check_args(gar_rule rule, int n, int f, int m) { return check_rule_args(rule, n, f, m); }

int gar_num_selected(gar_rule rule, int n, int f, int m) {
  if (check_rule_args(rule, n, f, m) != GAR_OK) return 0;
  if (rule == GAR_BULYAN) return n - 2 * f;
  return effective_m(rule, n, f, m);   // Krum 1, Multi-Krum m, MDA n - f
}

gar_status gar_aggregate_ex(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                            float* out, int32_t* indices_dev, void* workspace, size_t workspace_bytes,
                            gar_stream_t stream) {
  gar::OutPtrs none{};
  return aggregate_impl(rule, grads, n, f, m, d, out, none, indices_dev, workspace, workspace_bytes, stream);
}

gar_status gar_aggregate_bcast(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                               float* out, float* const* extra_outs, int n_extra, int32_t* indices_dev,
                               void* workspace, size_t workspace_bytes, gar_stream_t stream) {
  gar::OutPtrs extra{};
  gar_status s = make_extra(extra_outs, n_extra, &extra);
  if (s != GAR_OK) return s;
  return aggregate_impl(rule, grads, n, f, m, d, out, extra, indices_dev, workspace, workspace_bytes, stream);
}

gar_status gar_aggregate(gar_rule rule, const float* const* grads, int n, int f, int64_t d, float* out,
                         gar_stream_t stream) {
  gar_status s = check_rule_args(rule, n, f, 0);
  if (s != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* ws = nullptr;
  const size_t bytes = gar_workspace_bytes(rule, n, f, d);
  if (bytes) {
    if ((s = cuda_status(cudaMallocAsync(&ws, bytes, st))) != GAR_OK) return s;
  }
  s = gar_aggregate_ex(rule, grads, n, f, 0, d, out, nullptr, ws, bytes, stream);
  if (ws) {
    const gar_status f = cuda_status(cudaFreeAsync(ws, st));
    if (s == GAR_OK) s = f;
  }
  return s;
}

gar_status gar_select(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                      int32_t* indices_dev, int* n_selected_host, void* workspace, size_t workspace_bytes,
                      gar_stream_t stream) {
  return select_impl(rule, grads, n, f, m, d, indices_dev, n_selected_host, workspace, workspace_bytes, stream,
                     GAR_F32);
}

gar_status gar_distances(const float* const* grads, int n, int64_t d, double* D_dev, void* workspace,
                         size_t workspace_bytes, gar_stream_t stream) {
  return distances_impl(grads, n, d, D_dev, workspace, workspace_bytes, stream, GAR_F32);
}

gar_status gar_gram_partial(const float* const* grads, int n, int64_t d_local, double* gram_dev, void* workspace,
                            size_t workspace_bytes, gar_stream_t stream) {
  return gram_partial_impl(grads, n, d_local, gram_dev, workspace, workspace_bytes, stream, GAR_F32);
}

gar_status gar_select_from_gram(gar_rule rule, const double* gram_dev, int n, int f, int m, int32_t* indices_dev,
                                int* n_selected_host, void* workspace, size_t workspace_bytes,
                                gar_stream_t stream) {
  gar_status s = check_rule_args(rule, n, f, m);
  if (s != GAR_OK) return s;
  if (!is_krum_family(rule)) return GAR_ERR_UNSUPPORTED;
  if (!gram_dev || !indices_dev) return GAR_ERR_INVALID_ARGUMENT;
  // MDA needs the workspace (distance matrix + enumeration scratch); the
  // other rules run in one CTA's shared memory
  if (rule == GAR_MDA && (!workspace || workspace_bytes < ws_bytes_for(n))) return GAR_ERR_WORKSPACE;
  if ((s = check_device_ptr(gram_dev)) != GAR_OK) return s;
  if ((s = check_device_ptr(indices_dev)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int me = effective_m(rule, n, f, m);
  Workspace w{};
  if (workspace) w = carve(workspace, n);
  if ((s = run_select(rule, gram_dev, n, f, me, indices_dev, nullptr, workspace ? &w : nullptr, st)) != GAR_OK)
    return s;
  if (n_selected_host) *n_selected_host = gar_num_selected(rule, n, f, m);
  return GAR_OK;
}

gar_status gar_combine(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d_local,
                       const int32_t* indices_dev, float* out, gar_stream_t stream) {
  gar::OutPtrs none{};
  return combine_impl(rule, grads, n, f, m, d_local, indices_dev, out, none, stream);
}

gar_status gar_combine_bcast(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d_local,
                             const int32_t* indices_dev, float* out, float* const* extra_outs, int n_extra,
                             gar_stream_t stream) {
  gar::OutPtrs extra{};
  gar_status s = make_extra(extra_outs, n_extra, &extra);
  if (s != GAR_OK) return s;
  return combine_impl(rule, grads, n, f, m, d_local, indices_dev, out, extra, stream);
}

gar_status gar_aggregate_mcast(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                               float* out, float* out_mc, int32_t* indices_dev, void* workspace,
                               size_t workspace_bytes, gar_stream_t stream) {
  gar::OutPtrs extra{};
  gar_status s = make_mc(out_mc, &extra);
  if (s != GAR_OK) return s;
  return aggregate_impl(rule, grads, n, f, m, d, out, extra, indices_dev, workspace, workspace_bytes, stream);
}

gar_status gar_combine_mcast(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d_local,
                             const int32_t* indices_dev, float* out, float* out_mc, gar_stream_t stream) {
  gar::OutPtrs extra{};
  gar_status s = make_mc(out_mc, &extra);
  if (s != GAR_OK) return s;
  return combine_impl(rule, grads, n, f, m, d_local, indices_dev, out, extra, stream);
}

gar_status gar_aggregate_sgd(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                             float* params, float lr, int32_t* indices_dev, void* workspace, size_t workspace_bytes,
                             gar_stream_t stream) {
  if (!(lr == lr) || lr == INFINITY || lr == -INFINITY) return GAR_ERR_INVALID_ARGUMENT;
  gar::OutPtrs extra{};
  extra.sgd = 1;
  extra.lr = lr;
  return aggregate_impl(rule, grads, n, f, m, d, params, extra, indices_dev, workspace, workspace_bytes, stream);
}

gar_status gar_combine_sgd(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d_local,
                           const int32_t* indices_dev, float* params, float lr, gar_stream_t stream) {
  if (!(lr == lr) || lr == INFINITY || lr == -INFINITY) return GAR_ERR_INVALID_ARGUMENT;
  gar::OutPtrs extra{};
  extra.sgd = 1;
  extra.lr = lr;
  return combine_impl(rule, grads, n, f, m, d_local, indices_dev, params, extra, stream);
}

gar_status gar_gram_exchange(const float* const* grads, int n, int64_t d_local, double* const* peer_slots,
                             uint32_t* const* peer_flags, int rank, int world, uint32_t epoch, double* gram_dev,
                             float* const* stage_rows, void* workspace, size_t workspace_bytes,
                             gar_stream_t stream) {
  if (n < 1 || n > GAR_MAX_N || !gram_dev) return GAR_ERR_INVALID_ARGUMENT;
  if (world < 1 || world > gar::kMaxWorld || rank < 0 || rank >= world || !peer_slots || !peer_flags)
    return GAR_ERR_INVALID_ARGUMENT;
  gar::PeerSlots slots{};
  gar::PeerFlags flags{};
  for (int r = 0; r < world; ++r) {
    if (!peer_slots[r] || !peer_flags[r]) return GAR_ERR_INVALID_ARGUMENT;
    if ((reinterpret_cast<uintptr_t>(peer_slots[r]) & 7u) || (reinterpret_cast<uintptr_t>(peer_flags[r]) & 3u))
      return GAR_ERR_ALIGNMENT;
    slots.p[r] = peer_slots[r];
    flags.p[r] = peer_flags[r];
  }
  gar_status s = check_rows(grads, n, d_local);
  if (s != GAR_OK) return s;
  if (stage_rows && (s = check_rows(stage_rows, n, d_local)) != GAR_OK) return s;
  if (!workspace || workspace_bytes < ws_bytes_for(n)) return GAR_ERR_WORKSPACE;
  if ((s = check_device_rows(grads, n, nullptr)) != GAR_OK) return s;
  if ((s = check_device_ptr(gram_dev)) != GAR_OK) return s;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace w = carve(workspace, n);
  int parts = 0;
  if ((s = cuda_status(gar::launch_gram_partials(grads, n, d_local, w.partials, num_sms(), &parts, st,
                                                 stage_rows))) != GAR_OK)
    return s;
  return cuda_status(gar::launch_gram_exchange(w.partials, parts, n, slots, flags, world, rank, epoch, gram_dev, st));
}

gar_status gar_nonfinite_rows(const float* const* grads, int n, int64_t d, uint64_t* mask_dev,
                              gar_stream_t stream) {
  if (n < 1 || n > GAR_MAX_N || !mask_dev) return GAR_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(mask_dev) & 7u) return GAR_ERR_ALIGNMENT;
  gar_status s = check_rows(grads, n, d);
  if (s != GAR_OK) return s;
  if ((s = check_device_rows(grads, n, mask_dev)) != GAR_OK) return s;
  return cuda_status(gar::launch_nonfinite_rows(grads, n, d, mask_dev, num_sms(),
                                                reinterpret_cast<cudaStream_t>(stream)));
}

gar_status gar_trimmed_membership(const float* const* grads, int n, int f, int64_t d, uint64_t* mask_dev,
                                  gar_stream_t stream) {
  gar_status s = check_rule_args(GAR_TRIMMED_MEAN, n, f, 0);
  if (s != GAR_OK) return s;
  if ((s = check_rows(grads, n, d)) != GAR_OK) return s;
  if (!mask_dev) return GAR_ERR_INVALID_ARGUMENT;
  if (reinterpret_cast<uintptr_t>(mask_dev) & 7u) return GAR_ERR_ALIGNMENT;
  if ((s = check_device_rows(grads, n, mask_dev)) != GAR_OK) return s;
  return cuda_status(gar::launch_trimmed_membership(grads, n, f, d, mask_dev, num_sms(),
                                                    reinterpret_cast<cudaStream_t>(stream)));
}

// ---- bf16 gradient rows (R16) -------------------
gar_status gar_aggregate_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m, int64_t d,
                            float* out, int32_t* indices_dev, void* workspace, size_t workspace_bytes,
                            gar_stream_t stream) {
  gar::OutPtrs none{};
  return aggregate_impl(rule, rows_cast(grads), n, f, m, d, out, none, indices_dev, workspace, workspace_bytes,
                        stream, dtype);
}

gar_status gar_select_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m, int64_t d,
                         int32_t* indices_dev, int* n_selected_host, void* workspace, size_t workspace_bytes,
                         gar_stream_t stream) {
  return select_impl(rule, rows_cast(grads), n, f, m, d, indices_dev, n_selected_host, workspace, workspace_bytes,
                     stream, dtype);
}

gar_status gar_distances_dt(gar_dtype dtype, const void* const* grads, int n, int64_t d, double* D_dev,
                            void* workspace, size_t workspace_bytes, gar_stream_t stream) {
  return distances_impl(rows_cast(grads), n, d, D_dev, workspace, workspace_bytes, stream, dtype);
}

gar_status gar_gram_partial_dt(gar_dtype dtype, const void* const* grads, int n, int64_t d_local, double* gram_dev,
                               void* workspace, size_t workspace_bytes, gar_stream_t stream) {
  return gram_partial_impl(rows_cast(grads), n, d_local, gram_dev, workspace, workspace_bytes, stream, dtype);
}

gar_status gar_combine_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m,
                          int64_t d_local, const int32_t* indices_dev, float* out, gar_stream_t stream) {
  gar::OutPtrs none{};
  return combine_impl(rule, rows_cast(grads), n, f, m, d_local, indices_dev, out, none, stream, dtype);
}

}  // extern "C"
