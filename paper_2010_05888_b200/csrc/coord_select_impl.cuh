#pragma once
// coord_select_impl.cuh — the per-coordinate selection kernel (rows a1-a4, a8, a9 of
// DESIGN.md §1): Average, Median, trimmed mean, Multi-Krum/Krum combine and
// the Bulyan coordinate phase.  Product code for sm_100a.
//
// Dataflow (one persistent CTA per SM slot):
//   producer warp : one elected lane streams [R rows x T coords] tiles into a
//                   multi-stage shared-memory ring with 1D TMA bulk copies
//                   (cp.async.bulk ... mbarrier::complete_tx), L2 evict_first;
//   8 consumer warps: thread c owns column c of the tile, reads its R values
//                   from shared memory (conflict-free), canonicalises them
//                   (R1), runs a straight-line FMNMX network from
//                   networks.cuh, accumulates averages in fp64 (R2) and writes
//                   one coalesced fp32 per coordinate.
// HBM traffic is the algorithmic minimum: every input byte read once, every
// output byte written once.
#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "coord_select.h"
#include "networks.cuh"

namespace gar {

// W consumer warps (one coordinate per thread per tile) + kProducers producer
// warps.  W = 15 for up to 32 rows: 480-coordinate tiles = 1920 B per row per
// bulk copy, one CTA per SM with a ~180 KB ring; W = 7 above 32 rows keeps 3
// stages of 63 rows in shared memory.  Copy size AND the number of issuing
// warps matter: bulk-copy issue is limited per warp (tools/membench2.cu:
// 31 rows x 1 KB go 1.3 -> 5.5 TB/s from 1 to 8 issuing warps), so producer
// warp p issues rows r = p mod kProducers and arms its own stage barrier.
constexpr int kProducers = 4;
// Consumer warps per CTA (one CTA per SM).  The trimmed mean and the Bulyan
// phase are ALU-bound (FMNMX networks) and gain from more warps to overlap: 24
// warps (2 stages of 95 KB at 31 rows) run the C3 trimmed mean in 0.62 ms
// against 0.69 with 15, and C3 Bulyan in 0.99 against 1.035; the Median, at
// HBM speed, is best with 15 (3 stages).  Above 32 rows 12 warps (2 stages of
// <= 98 KB): the Median of 63 in 1.16 ms against 1.43 with 7 and 1.40 with
// direct loads; the trimmed mean takes 16 at 33..48 rows (n = 39: 0.85 ms
// against 0.93 with direct loads).  Measured in profiles/r1_loader_choice.md.
template <int MODE, int N>
constexpr int consumer_warps() {
  if constexpr (N > 48) return 12;
  if constexpr (N > 32) return MODE == kModeTrimmed ? 16 : 12;
  return (MODE == kModeTrimmed || MODE == kModeBulyan) ? 24 : 15;
}

struct CoordParams {
  RowPtrs rows;
  const int32_t* idx;   // nullptr: rows 0..R-1; else R selected input indices
  float* out;
  OutPtrs extra;        // further destinations of every result (peer GPUs' buffers)
  int64_t d;
  int R;                // rows consumed per coordinate
  int f;                // trimmed mean: trim per side; Bulyan: declared f
  int stages;
  int l2_hint;          // 1: bulk copies carry an L2 evict-first policy
  int64_t num_tiles;
};

// ---------------------------------------------------------------- per-mode math
// Average over R values in index order, fp64 (R2).  The additions stay in
// index order (bit-exact against the oracle even when the fp64 sum rounds);
// loads and conversions are batched 8 at a time ahead of the dependent DADD
// chain so it is not serialised behind LDS/F2F latency.
__device__ __forceinline__ float avg_column(const float* col, int R, int stride) {
  double s = 0.0;
  int i = 0;
  for (; i + 8 <= R; i += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = static_cast<double>(col[(i + u) * stride]);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < R; ++i) s += static_cast<double>(col[i * stride]);
  return static_cast<float>(s / R);
}

// The networks take the raw values: their compare-exchange (fminf + max.NaN,
// networks.cuh) moves a NaN exactly like +inf, so only the outputs a rule
// uses are mapped NaN -> +inf.  -0 and +0 compare equal, which can only swap
// zeros; zeros add exactly nothing to an fp64 sum that starts at +0; and
// Bulyan's closeness |y - med| and its value comparisons treat -0 == +0.
// The median output is canonicalised (R1), so every result equals that of
// the canonical inputs.
__device__ __forceinline__ float nan_to_inf(float v) { return fminf(v, __int_as_float(0x7f800000)); }

template <int N>
__device__ __forceinline__ float median_column(float* v) {
  gar_net::median_net<N>(v);
  if constexpr (N % 2 == 1) {
    return canon(v[(N - 1) / 2]);
  } else {
    return static_cast<float>((static_cast<double>(canon(v[N / 2 - 1])) + static_cast<double>(canon(v[N / 2]))) *
                              0.5);
  }
}

// fp64 sum of v[F], ..., v[N-F-1] in ascending order (R2), F a compile-time
// constant so only the kept values are converted and added.
template <int N, int F>
__device__ __forceinline__ double sum_kept(const float* v, int f) {
  if constexpr (2 * F >= N) {
    return 0.0;
  } else {
    if (f != F) return sum_kept<N, F + 1>(v, f);
    double s = 0.0;
#pragma unroll
    for (int t = F; t < N - F; ++t) s += static_cast<double>(nan_to_inf(v[t]));
    return s;
  }
}

// At the paper's f for n = 4f + 3 (every BASELINE configuration) a
// network pruned to the kept positions (gar_net::trim_net, ~10% fewer
// min/max than the full sort); any other f takes the full sort.
template <int N>
__device__ __forceinline__ float trimmed_column(float* v, int f) {
  constexpr int F = gar_net::trim_f<N>();
  double s;
  if (f == F) {
    gar_net::trim_net<N>(v);
    s = sum_kept<N, F>(v, f);
  } else {
    gar_net::sort_net<N>(v);
    s = sum_kept<N, 0>(v, f);
  }
  return static_cast<float>(s / (N - 2 * f));
}

__device__ __forceinline__ float closeness(float y, float med) {
  return (y == med) ? 0.0f : fabsf(__fsub_rn(y, med));
}

// Bulyan coordinate phase over THETA values (NaN -> +inf; zeros of either sign) (positions = ascending
// input index).  Keeps the beta = THETA - 2f values with the smallest
// (closeness, index) (R8) and averages them in ascending order (R2).
//
// In value-sorted order the kept multiset is a window [s*, s*+beta): closeness
// decreases towards the median from the left and increases from the right, so
// "shift the window right by one" (drop v[s], take v[s+beta]) is a monotone
// predicate and s* = s_min + #{s : c(v[s+beta]) < c(v[s])}.  A closeness tie
// between two DIFFERENT values needs the input indices: those (rare) columns
// take the exact rank-count path over the index-ordered values.
// The sorted column is parked in the CTA's shared-memory slot so the
// runtime-offset reads (beta depends on the runtime f) are plain LDS.
template <int THETA>
__device__ __forceinline__ float bulyan_column(float* v, float* col, int stride, int f,
                                               const float* const* rowp, int64_t gidx) {
  const int beta = THETA - 2 * f;
  gar_net::sort_net<THETA>(v);
#pragma unroll
  for (int t = 0; t < THETA; ++t) {
    v[t] = nan_to_inf(v[t]);
    col[t * stride] = v[t];
  }
  constexpr int h = (THETA - 1) / 2;
  float med;
  if constexpr (THETA % 2 == 1) {
    med = v[h];
  } else {
    med = static_cast<float>((static_cast<double>(v[h]) + static_cast<double>(v[h + 1])) * 0.5);
  }
  constexpr int h_hi = (THETA % 2 == 1) ? h : h + 1;
  const int s_min = max(0, h - beta + 1);
  const int s_max = min(THETA - beta, h_hi);
  int shift = 0;
  bool tie = false;
  for (int s = s_min; s < s_max; ++s) {
    const float left = col[s * stride], right = col[(s + beta) * stride];
    const float cl = closeness(left, med), cr = closeness(right, med);
    shift += (cr < cl) ? 1 : 0;
    tie |= (cr == cl) && (right != left);
  }
  int start = s_min + shift;
  if (tie) {
    // exact path: kept_t  <=>  #{u : (c_u, u) < (c_t, t)} < beta, index order
    int p = 0, kL = 0;
    for (int t = 0; t < THETA; ++t) {
      const float yt = canon(__ldg(rowp[t] + gidx));
      const float ct = closeness(yt, med);
      int rank = 0;
      for (int u = 0; u < THETA; ++u) {
        const float cu = closeness(canon(__ldg(rowp[u] + gidx)), med);
        rank += (cu < ct || (cu == ct && u < t)) ? 1 : 0;
      }
      p += (yt < med) ? 1 : 0;
      kL += (rank < beta && yt < med) ? 1 : 0;
    }
    start = p - kL;
  }
  double acc = 0.0;
  for (int j = 0; j < beta; ++j) acc += static_cast<double>(col[(start + j) * stride]);
  return static_cast<float>(acc / beta);
}

// Bulyan coordinate phase when beta = 3, i.e. f = (THETA-3)/2 (n = 4f + 3,
// P:556; every BASELINE configuration), THETA odd >= 5.  The kept window
// starts at h-2, h-1 or h (it holds the median itself, closeness 0), so a
// network that sorts only positions h-2..h+2 suffices and the window stays in
// registers.  A closeness tie between two different values takes the exact
// definition: the beta values of smallest (closeness, index) over the
// index-ordered canonical inputs, summed in ascending order.
template <int THETA>
__device__ __forceinline__ float bulyan_column_b3(float* v, const float* const* rowp, int64_t gidx) {
  static_assert(THETA % 2 == 1 && THETA >= 5, "beta = 3 window");
  constexpr int h = (THETA - 1) / 2;
  gar_net::window_net<THETA>(v);
  const float a0 = nan_to_inf(v[h - 2]), a1 = nan_to_inf(v[h - 1]), med = nan_to_inf(v[h]);
  const float a3 = nan_to_inf(v[h + 1]), a4 = nan_to_inf(v[h + 2]);
  const float c0 = closeness(a0, med), c1 = closeness(a1, med);
  const float c3 = closeness(a3, med), c4 = closeness(a4, med);
  const int shift = ((c3 < c0) ? 1 : 0) + ((c4 < c1) ? 1 : 0);
  const bool tie = (c3 == c0 && a3 != a0) || (c4 == c1 && a4 != a1);
  float k0, k1, k2;
  if (!tie) {
    k0 = shift == 0 ? a0 : (shift == 1 ? a1 : med);
    k1 = shift == 0 ? a1 : (shift == 1 ? med : a3);
    k2 = shift == 0 ? med : (shift == 1 ? a3 : a4);
  } else {
    float kept[3] = {0.f, 0.f, 0.f};
    int nk = 0;
    for (int t = 0; t < THETA; ++t) {
      const float yt = canon(__ldg(rowp[t] + gidx));
      const float ct = closeness(yt, med);
      int rank = 0;
      for (int u = 0; u < THETA; ++u) {
        const float cu = closeness(canon(__ldg(rowp[u] + gidx)), med);
        rank += (cu < ct || (cu == ct && u < t)) ? 1 : 0;
      }
      if (rank < 3 && nk < 3) kept[nk++] = yt;
    }
    k0 = fminf(kept[0], kept[1]);
    k1 = fmaxf(kept[0], kept[1]);
    k2 = fmaxf(k1, kept[2]);
    k1 = fminf(k1, kept[2]);
    const float lo = fminf(k0, k1);
    k1 = fmaxf(k0, k1);
    k0 = lo;
  }
  double acc = 0.0;
  acc += static_cast<double>(k0);
  acc += static_cast<double>(k1);
  acc += static_cast<double>(k2);
  return static_cast<float>(acc / 3);
}

template <int THETA>
__device__ __forceinline__ float bulyan_dispatch(float* v, float* col, int stride, int f,
                                                 const float* const* rowp, int64_t gidx) {
  if constexpr (THETA % 2 == 1 && THETA >= 5) {
    if (f == (THETA - 3) / 2) return bulyan_column_b3<THETA>(v, rowp, gidx);
  }
  return bulyan_column<THETA>(v, col, stride, f, rowp, gidx);
}

// ---------------------------------------------------------------- the kernel
template <int MODE, int N, int W>
__global__ void __launch_bounds__(32 * (W + kProducers), 1) coord_select_kernel(const __grid_constant__ CoordParams p) {
  constexpr int kConsumerWarps = W;
  constexpr int kTile = 32 * W;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int R = (N > 0) ? N : p.R;
  const int stages = p.stages;
  float* tiles = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(stages) * R * kTile * sizeof(float));  // [stages][kProducers]
  uint64_t* empty = full + stages * kProducers;
  __shared__ const float* rowp[GAR_MAX_N];
  __shared__ int sel_s[GAR_MAX_N];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    if (p.idx) {
      // selected rows in ascending input-index order (R2, R8 tie order)
      for (int r = 0; r < R; ++r) {
        int v = p.idx[r], t = r;
        while (t > 0 && sel_s[t - 1] > v) { sel_s[t] = sel_s[t - 1]; --t; }
        sel_s[t] = v;
      }
      for (int r = 0; r < R; ++r) rowp[r] = p.rows.p[sel_s[r]];
    } else {
      for (int r = 0; r < R; ++r) rowp[r] = p.rows.p[r];
    }
    for (int s = 0; s < stages; ++s) {
      for (int q = 0; q < kProducers; ++q) mbar_init(&full[s * kProducers + q], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t d = p.d;
  if (warp >= kConsumerWarps) {
    // ------------------------------------------------ producers (TMA bulk)
    const int q = warp - kConsumerWarps;           // rows r = q (mod kProducers)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int my_rows = (R > q) ? (R - q + kProducers - 1) / kProducers : 0;
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
        mbar_wait(&empty[stage], phase ^ 1);
        const int64_t start = tile * kTile;
        const int cnt = static_cast<int>((d - start < kTile ? d - start : int64_t(kTile)));
        const uint32_t bytes = static_cast<uint32_t>(cnt & ~3) * 4u;
        uint64_t* bar = &full[stage * kProducers + q];
        mbar_arrive_expect_tx(bar, bytes * my_rows);
        if (bytes) {
          float* dst = tiles + size_t(stage) * R * kTile;
          if (p.l2_hint) {
            for (int r = q; r < R; r += kProducers) bulk_g2s(dst + r * kTile, rowp[r] + start, bytes, bar, pol);
          } else {
            for (int r = q; r < R; r += kProducers) bulk_g2s_plain(dst + r * kTile, rowp[r] + start, bytes, bar);
          }
        }
        if (++stage == stages) { stage = 0; phase ^= 1; }
      }
    }
    return;
  }

  // -------------------------------------------------- consumers
  int stage = 0;
  uint32_t phase = 0;
  const int c = threadIdx.x;
  for (int64_t tile = blockIdx.x; tile < p.num_tiles; tile += gridDim.x) {
#pragma unroll
    for (int q = 0; q < kProducers; ++q) mbar_wait(&full[stage * kProducers + q], phase);
    const int64_t start = tile * kTile;
    const int cnt = static_cast<int>((d - start < kTile ? d - start : int64_t(kTile)));
    const int bulk_cnt = cnt & ~3;
    float* col = tiles + size_t(stage) * R * kTile + c;
    if (c >= bulk_cnt && c < cnt) {
      // ragged tail (< 4 coordinates): not bulk-copied, fetch directly
      for (int r = 0; r < R; ++r) col[r * kTile] = __ldg(rowp[r] + start + c);
    }
    if (c < cnt) {
      // fused server step: the parameter is loaded before the column work so
      // its latency overlaps it
      const float pv = p.extra.sgd ? __ldcs(p.out + start + c) : 0.0f;
      float res;
      if constexpr (MODE == kModeAverage) {
        res = avg_column(col, R, kTile);
      } else {
        float v[N > 0 ? N : 1];
#pragma unroll
        for (int r = 0; r < N; ++r) v[r] = col[r * kTile];
        if constexpr (MODE == kModeMedian) {
          res = median_column<N>(v);
        } else if constexpr (MODE == kModeTrimmed) {
          res = trimmed_column<N>(v, p.f);
        } else {
          res = bulyan_dispatch<N>(v, col, kTile, p.f, rowp, start + c);
        }
      }
      store_result(p.out, p.extra, start + c, res, pv);
    }
    // generic-proxy writes into the ring (the ragged-tail fill, Bulyan's sorted
    // column park) must be ordered before the producer's next async-proxy
    // (bulk copy) overwrite of this stage: PTX memory model, ADVICE r1
    if (MODE == kModeBulyan || (c >= bulk_cnt && c < cnt)) fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == stages) { stage = 0; phase ^= 1; }
  }
}

// ---------------------------------------------------------------- LDG variant
// Direct-load variant: thread = coordinate, its R values are loaded straight into
// registers (coalesced 128 B per warp and row, streaming), no staging.  The
// register file (256 KB/SM) holds more in-flight data than the shared-memory
// ring, which matters for large R (tools/membench.cu: ~6.5 TB/s at any R with
// >= 32 warps/SM).  Bulyan's runtime-offset window reads use a per-thread
// shared-memory column.
constexpr int kLdgThreads = 256;

template <int MODE, int N>
__device__ __forceinline__ void coord_ldg_body(const CoordParams& p, const float** rowp, int* sel_s) {
  extern __shared__ __align__(16) unsigned char ldg_smem[];
  const int R = (N > 0) ? N : p.R;
  if (threadIdx.x == 0) {
    if (p.idx) {
      for (int r = 0; r < R; ++r) {
        int v = p.idx[r], t = r;
        while (t > 0 && sel_s[t - 1] > v) { sel_s[t] = sel_s[t - 1]; --t; }
        sel_s[t] = v;
      }
      for (int r = 0; r < R; ++r) rowp[r] = p.rows.p[sel_s[r]];
    } else {
      for (int r = 0; r < R; ++r) rowp[r] = p.rows.p[r];
    }
  }
  __syncthreads();
  const int64_t d = p.d;
  const int64_t step = int64_t(gridDim.x) * kLdgThreads;
#ifndef GAR_LDG_PREFETCH_MAX_N
#define GAR_LDG_PREFETCH_MAX_N 47
#endif
  if constexpr (MODE != kModeAverage && N > 0 && N <= GAR_LDG_PREFETCH_MAX_N) {
    // software pipeline: the next column's N loads are in flight while this
    // column goes through the network.  Up to 47 rows the kernel stays within
    // 128 registers (2+ CTAs per SM); measured 1-7 % faster for n = 11..47
    // and 5-6 % slower at n = 63 (171 registers), profiles/r1_sweep_C5.md.
    // Two register sets used alternately instead of the copy: more registers,
    // measured slower at every n.
    auto column = [&](float* v, int64_t k) {
      const float pv = p.extra.sgd ? __ldcs(p.out + k) : 0.0f;
      float res;
      if constexpr (MODE == kModeMedian) {
        res = median_column<N>(v);
      } else if constexpr (MODE == kModeTrimmed) {
        res = trimmed_column<N>(v, p.f);
      } else {
        float* col = reinterpret_cast<float*>(ldg_smem) + threadIdx.x;
        res = bulyan_dispatch<N>(v, col, kLdgThreads, p.f, rowp, k);
      }
      store_result(p.out, p.extra, k, res, pv);
    };
    auto load = [&](float* v, int64_t k) {
#pragma unroll
      for (int r = 0; r < N; ++r) v[r] = __ldcs(rowp[r] + k);
    };
    int64_t k = int64_t(blockIdx.x) * kLdgThreads + threadIdx.x;
    float v[N];
    if (k < d) load(v, k);
    for (; k < d; k += step) {
      const int64_t kn = k + step;
      float vn[N];
      if (kn < d) load(vn, kn);
      column(v, k);
#pragma unroll
      for (int r = 0; r < N; ++r) v[r] = vn[r];
    }
    return;
  }
  for (int64_t k = int64_t(blockIdx.x) * kLdgThreads + threadIdx.x; k < d; k += step) {
    const float pv = p.extra.sgd ? __ldcs(p.out + k) : 0.0f;     // fused server step (see above)
    float res;
    if constexpr (MODE == kModeAverage) {
      double s = 0.0;
      int i = 0;
      for (; i + 16 <= R; i += 16) {
        float v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcs(rowp[i + u] + k);
#pragma unroll
        for (int u = 0; u < 16; ++u) s += static_cast<double>(v[u]);
      }
      for (; i < R; ++i) s += static_cast<double>(__ldcs(rowp[i] + k));
      res = static_cast<float>(s / R);
    } else {
      float v[N];
#pragma unroll
      for (int r = 0; r < N; ++r) v[r] = __ldcs(rowp[r] + k);
      if constexpr (MODE == kModeMedian) {
        res = median_column<N>(v);
      } else if constexpr (MODE == kModeTrimmed) {
        res = trimmed_column<N>(v, p.f);
      } else {
        float* col = reinterpret_cast<float*>(ldg_smem) + threadIdx.x;
        res = bulyan_dispatch<N>(v, col, kLdgThreads, p.f, rowp, k);
      }
    }
    store_result(p.out, p.extra, k, res, pv);
  }
}

template <int MODE, int N>
__global__ void __launch_bounds__(kLdgThreads) coord_ldg_kernel(const __grid_constant__ CoordParams p) {
  __shared__ const float* rowp[GAR_MAX_N];
  __shared__ int sel_s[GAR_MAX_N];
  coord_ldg_body<MODE, N>(p, rowp, sel_s);
}

template <int MODE, int N>
inline cudaError_t launch_ldg(const CoordLaunch& L, cudaStream_t stream) {
  CoordParams p;
  for (int i = 0; i < GAR_MAX_N; ++i) p.rows.p[i] = (i < L.n) ? L.rows[i] : nullptr;
  p.idx = L.idx;
  p.out = L.out;
  p.extra = L.extra;
  p.d = L.d;
  p.R = L.R;
  p.f = L.f;
  p.stages = 0;
  p.l2_hint = 0;
  p.num_tiles = 0;
  const size_t smem = (MODE == kModeBulyan) ? size_t(L.R) * kLdgThreads * sizeof(float) : 0;
  auto kern = coord_ldg_kernel<MODE, N>;
  int occ = 0;
  cudaError_t e = cached_occupancy(kern, kLdgThreads, smem, &occ);
  if (e != cudaSuccess) return e;
  int64_t grid = int64_t(L.num_sms) * occ;
  const int64_t need = (L.d + kLdgThreads - 1) / kLdgThreads;
  if (grid > need) grid = need > 0 ? need : 1;
  kern<<<static_cast<unsigned>(grid), kLdgThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

// Loader selection (measured on B200, tools/ab_step.py, profiles/r1_loader_choice.md):
// the TMA ring (4 issuing warps) for the Median at every row count, for averages
// at 17..32 and 48..64 rows, the trimmed mean above 12 rows, the Bulyan phase
// at 17..32 rows; direct loads elsewhere.  GAR_COORD_LOADER=tma|ldg forces one.
// Returns 1 for LDG.
int coord_loader_ldg(int mode, int R);

// ---------------------------------------------------------------- host side
template <int MODE, int N, int W>
inline cudaError_t launch_mode_w(const CoordLaunch& L, cudaStream_t stream) {
  constexpr int kTile = 32 * W;
  constexpr int kThreads = 32 * (W + kProducers);
  CoordParams p;
  for (int i = 0; i < GAR_MAX_N; ++i) p.rows.p[i] = (i < L.n) ? L.rows[i] : nullptr;
  p.idx = L.idx;
  p.out = L.out;
  p.extra = L.extra;
  p.d = L.d;
  p.R = L.R;
  p.f = L.f;
  const size_t stage_bytes = size_t(L.R) * kTile * sizeof(float);
  int stages = static_cast<int>((200 * 1024) / stage_bytes);
  stages = max(2, min(8, stages));
  p.stages = stages;
  p.l2_hint = l2_evict_first_enabled();
  p.num_tiles = (L.d + kTile - 1) / kTile;
  const size_t smem = stages * stage_bytes + (kProducers + 1) * stages * sizeof(uint64_t);
  auto kern = coord_select_kernel<MODE, N, W>;
  int occ = 0;
  cudaError_t e = cached_occupancy(kern, kThreads, smem, &occ);
  if (e != cudaSuccess) return e;
  int64_t grid = int64_t(L.num_sms) * occ;
  if (grid > p.num_tiles) grid = p.num_tiles > 0 ? p.num_tiles : 1;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

template <int MODE, int N>
inline cudaError_t launch_mode(const CoordLaunch& L, cudaStream_t stream) {
  if (coord_loader_ldg(MODE, L.R)) return launch_ldg<MODE, N>(L, stream);
  if constexpr (N > 0) {
    return launch_mode_w<MODE, N, consumer_warps<MODE, N>()>(L, stream);
  } else {
    if (L.R <= 32) return launch_mode_w<MODE, 0, 15>(L, stream);
    return launch_mode_w<MODE, 0, 7>(L, stream);
  }
}

template <int MODE, int LO, int HI>
inline cudaError_t dispatch_range(const CoordLaunch& L, cudaStream_t stream) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (L.R == LO) return launch_mode<MODE, LO>(L, stream);
    return dispatch_range<MODE, LO + 1, HI>(L, stream);
  }
}

}  // namespace gar
