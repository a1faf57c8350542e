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
#include <type_traits>

#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "networks.cuh"

// A/B knobs (defaults = product): consumer warps of the Bulyan phase up to 32
// rows, and the TMA ring budget in KB
#ifndef GAR_BULYAN_W
#define GAR_BULYAN_W 24
#endif
#ifndef GAR_RING_KB
#define GAR_RING_KB 200
#endif

namespace gar {

// W consumer warps (one coordinate per thread per tile) + kProducers producer
// warps.  W = 15 for up to 32 rows: 480-coordinate tiles = 1920 B per row per
// bulk copy, one CTA per SM with a ~180 KB ring; W = 7 above 32 rows keeps 3
// stages of 63 rows in shared memory.  Copy size AND the number of issuing
// warps matter: bulk-copy issue is limited per warp (tools/membench2.cu:
// 31 rows x 1 KB go 1.3 -> 5.5 TB/s from 1 to 8 issuing warps), so producer
// warp p issues rows r = p mod kProducers; each arms the stage's one "full"
// barrier (kProducers arrivals, each with its own expected bytes), so a
// consumer waits on one barrier per tile.
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
  if constexpr (MODE == kModeBulyan) return GAR_BULYAN_W;
  return MODE == kModeTrimmed ? 24 : 15;
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
// Each function takes the R (or N) values of one thread-element column: one
// coordinate for T = float, two adjacent coordinates for T = bf2 (elem.cuh),
// and writes res[h] for h < Elem<T>::EPT.  val(x, h) is the exact fp32 value
// of half h; every rule below is the fp32 definition on those values (R16).
__device__ __forceinline__ float val(float x, int) { return x; }
__device__ __forceinline__ float val(bf2 x, int h) { return bf_half(x, h); }

// Average over R values in index order, fp64 (R2).  The additions stay in
// index order (bit-exact against the oracle even when the fp64 sum rounds);
// loads and conversions are batched 8 at a time ahead of the dependent DADD
// chain so it is not serialised behind LDS/F2F latency.
__device__ __forceinline__ void avg_column(const float* col, int R, int stride, float* res) {
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
  res[0] = static_cast<float>(s / R);
}

__device__ __forceinline__ void avg_column(const bf2* col, int R, int stride, float* res) {
  double s0 = 0.0, s1 = 0.0;
  int i = 0;
  for (; i + 8 <= R; i += 8) {
    bf2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = col[(i + u) * stride];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s0 += static_cast<double>(bf_lo(v[u]));
      s1 += static_cast<double>(bf_hi(v[u]));
    }
  }
  for (; i < R; ++i) {
    const bf2 v = col[i * stride];
    s0 += static_cast<double>(bf_lo(v));
    s1 += static_cast<double>(bf_hi(v));
  }
  res[0] = static_cast<float>(s0 / R);
  res[1] = static_cast<float>(s1 / R);
}

// The networks take the raw values: their compare-exchange (vmin + vmax_nan,
// networks.cuh / elem.cuh) moves a NaN exactly like +inf, so only the outputs
// a rule uses are mapped NaN -> +inf.  -0 and +0 compare equal, which can only
// swap zeros; zeros add exactly nothing to an fp64 sum that starts at +0; and
// Bulyan's closeness |y - med| and its value comparisons treat -0 == +0.
// The median output is canonicalised (R1), so every result equals that of
// the canonical inputs.
__device__ __forceinline__ float nan_to_inf(float v) { return fminf(v, __int_as_float(0x7f800000)); }
__device__ __forceinline__ bf2 nan_to_inf(bf2 v) { return vmin(v, bf2{0x7f807f80u}); }

template <int N, class T>
__device__ __forceinline__ void median_column(T* v, float* res) {
  gar_net::median_net<N>(v);
#pragma unroll
  for (int h = 0; h < Elem<T>::EPT; ++h) {
    if constexpr (N % 2 == 1) {
      res[h] = canon(val(v[(N - 1) / 2], h));
    } else {
      res[h] = static_cast<float>(
          (static_cast<double>(canon(val(v[N / 2 - 1], h))) + static_cast<double>(canon(val(v[N / 2], h)))) * 0.5);
    }
  }
}

// fp64 sum of v[F], ..., v[N-F-1] (half h) in ascending order (R2), F a
// compile-time constant so only the kept values are converted and added.
// The kept values are summed raw: a NaN among them stands for +inf (R1), and
// a raw sum is NaN exactly when the canonical one is +inf or NaN, so one
// fix-up replaces the per-value NaN -> +inf mapping: NaN -> +inf unless the
// smallest kept value is -inf (then the canonical sum is -inf + inf = NaN).
template <int N, int F, class T>
__device__ __forceinline__ double sum_kept(const T* v, int f, int h) {
  if constexpr (2 * F >= N) {
    return 0.0;
  } else {
    if (f != F) return sum_kept<N, F + 1>(v, f, h);
    double s = 0.0;
#pragma unroll
    for (int t = F; t < N - F; ++t) s += static_cast<double>(val(v[t], h));
    if (s != s) s = (val(v[F], h) == -__int_as_float(0x7f800000)) ? s : static_cast<double>(__int_as_float(0x7f800000));
    return s;
  }
}

// At the paper's f for n = 4f + 3 (every BASELINE configuration) a
// network pruned to the kept positions (gar_net::trim_net, ~10% fewer
// min/max than the full sort); any other f takes the full sort.
template <int N, class T>
__device__ __forceinline__ void trimmed_column(T* v, int f, float* res) {
  constexpr int F = gar_net::trim_f<N>();
  const bool pruned = (f == F);
  if (pruned) {
    gar_net::trim_net<N>(v);
  } else {
    gar_net::sort_net<N>(v);
  }
#pragma unroll
  for (int h = 0; h < Elem<T>::EPT; ++h) {
    const double s = pruned ? sum_kept<N, F>(v, f, h) : sum_kept<N, 0>(v, f, h);
    res[h] = static_cast<float>(s / (N - 2 * f));
  }
}

__device__ __forceinline__ float closeness(float y, float med) {
  return (y == med) ? 0.0f : fabsf(__fsub_rn(y, med));
}

// Exact definition of Bulyan's kept set (R8), for the rare columns with a
// closeness tie between two DIFFERENT values: the beta values of smallest
// (closeness, input index) over the index-ordered canonical inputs of
// coordinate gidx, read straight from the rows.  Returns the start of the
// kept window in value-sorted order (p - kL: values below the median minus
// the kept ones below it).
template <class T>
__device__ __forceinline__ int bulyan_exact_start(int theta, int beta, float med, const float* const* rowp,
                                                  int64_t gidx) {
  int p = 0, kL = 0;
  for (int t = 0; t < theta; ++t) {
    const float yt = canon(Elem<T>::value(rowp[t], gidx));
    const float ct = closeness(yt, med);
    int rank = 0;
    for (int u = 0; u < theta; ++u) {
      const float cu = closeness(canon(Elem<T>::value(rowp[u], gidx)), med);
      rank += (cu < ct || (cu == ct && u < t)) ? 1 : 0;
    }
    p += (yt < med) ? 1 : 0;
    kL += (rank < beta && yt < med) ? 1 : 0;
  }
  return p - kL;
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
template <int THETA, class T>
__device__ __forceinline__ void bulyan_column(T* v, T* col, int stride, int f, const float* const* rowp,
                                              int64_t gidx, float* res) {
  const int beta = THETA - 2 * f;
  gar_net::sort_net<THETA>(v);
#pragma unroll
  for (int t = 0; t < THETA; ++t) col[t * stride] = nan_to_inf(v[t]);
  constexpr int hm = (THETA - 1) / 2;
  constexpr int h_hi = (THETA % 2 == 1) ? hm : hm + 1;
  const int s_min = max(0, hm - beta + 1);
  const int s_max = min(THETA - beta, h_hi);
#pragma unroll
  for (int h = 0; h < Elem<T>::EPT; ++h) {
    float med;
    if constexpr (THETA % 2 == 1) {
      med = val(col[hm * stride], h);
    } else {
      med = static_cast<float>((static_cast<double>(val(col[hm * stride], h)) +
                                static_cast<double>(val(col[(hm + 1) * stride], h))) * 0.5);
    }
    int shift = 0;
    bool tie = false;
    for (int s = s_min; s < s_max; ++s) {
      const float left = val(col[s * stride], h), right = val(col[(s + beta) * stride], h);
      const float cl = closeness(left, med), cr = closeness(right, med);
      shift += (cr < cl) ? 1 : 0;
      tie |= (cr == cl) && (right != left);
    }
    const int start = tie ? bulyan_exact_start<T>(THETA, beta, med, rowp, gidx + h) : s_min + shift;
    double acc = 0.0;
    for (int j = 0; j < beta; ++j) acc += static_cast<double>(val(col[(start + j) * stride], h));
    res[h] = static_cast<float>(acc / beta);
  }
}

// The exact beta = 3 kept set of one coordinate (R8): the 3 values of
// smallest (closeness, input index), by one scan of the canonical inputs in
// index order that keeps the 3 best keys (a later index never displaces an
// equal closeness), then summed in ascending order.  The values come from the
// index-ordered raw column in shared memory (col, half h) when the caller has
// one, else from the rows in global memory.  O(THETA): bf16 inputs, with 8
// significant bits, tie often (med - a == b - med), so this path is not rare.
template <int THETA, class T>
__device__ __forceinline__ float bulyan_b3_exact(float med, const T* col, int stride, int h, const float* const* rowp,
                                              int64_t gidx) {
  // keys: closeness bits (non-negative floats order like their bits; never
  // NaN here), sentinel above +inf
  uint32_t q0 = 0xFFFFFFFFu, q1 = 0xFFFFFFFFu, q2 = 0xFFFFFFFFu;
  float v0 = 0.f, v1 = 0.f, v2 = 0.f;
  for (int u = 0; u < THETA; ++u) {
    const float y = canon(col ? val(col[u * stride], h) : Elem<T>::value(rowp[u], gidx));
    const uint32_t q = __float_as_uint(closeness(y, med));
    if (q < q2) {
      if (q < q1) {
        q2 = q1; v2 = v1;
        if (q < q0) { q1 = q0; v1 = v0; q0 = q; v0 = y; } else { q1 = q; v1 = y; }
      } else {
        q2 = q; v2 = y;
      }
    }
  }
  const float kv[3] = {v0, v1, v2};
  float k0 = fminf(kv[0], kv[1]), k1 = fmaxf(kv[0], kv[1]);
  const float k2 = fmaxf(k1, kv[2]);
  k1 = fminf(k1, kv[2]);
  const float lo = fminf(k0, k1);
  k1 = fmaxf(k0, k1);
  k0 = lo;
  double acc = 0.0;
  acc += static_cast<double>(k0);
  acc += static_cast<double>(k1);
  acc += static_cast<double>(k2);
  return static_cast<float>(acc / 3);
}

// Bulyan coordinate phase when beta = 3, i.e. f = (THETA-3)/2 (n = 4f + 3,
// P:556; every BASELINE configuration), THETA odd >= 5.  The kept window
// starts at h-2, h-1 or h (it holds the median itself, closeness 0), so a
// network that sorts only positions h-2..h+2 suffices and the window stays in
// registers.  A closeness tie between two different values takes the exact
// definition (bulyan_b3_exact).
template <int THETA, class T>
__device__ __forceinline__ void bulyan_column_b3(T* v, const T* col, int stride, const float* const* rowp,
                                                 int64_t gidx, float* res) {
  static_assert(THETA % 2 == 1 && THETA >= 5, "beta = 3 window");
  constexpr int hm = (THETA - 1) / 2;
  gar_net::window_net<THETA>(v);
#pragma unroll
  for (int h = 0; h < Elem<T>::EPT; ++h) {
    const float a0 = nan_to_inf(val(v[hm - 2], h)), a1 = nan_to_inf(val(v[hm - 1], h));
    const float med = nan_to_inf(val(v[hm], h));
    const float a3 = nan_to_inf(val(v[hm + 1], h)), a4 = nan_to_inf(val(v[hm + 2], h));
    const float c0 = closeness(a0, med), c1 = closeness(a1, med);
    const float c3 = closeness(a3, med), c4 = closeness(a4, med);
    const int shift = ((c3 < c0) ? 1 : 0) + ((c4 < c1) ? 1 : 0);
    const bool tie = (c3 == c0 && a3 != a0) || (c4 == c1 && a4 != a1);
    if (tie) {
      res[h] = bulyan_b3_exact<THETA>(med, col, stride, h, rowp, gidx + h);
      continue;
    }
    const float k0 = shift == 0 ? a0 : (shift == 1 ? a1 : med);
    const float k1 = shift == 0 ? a1 : (shift == 1 ? med : a3);
    const float k2 = shift == 0 ? med : (shift == 1 ? a3 : a4);
    double acc = 0.0;
    acc += static_cast<double>(k0);
    acc += static_cast<double>(k1);
    acc += static_cast<double>(k2);
    res[h] = static_cast<float>(acc / 3);
  }
}

// RAWCOL: col holds this coordinate's raw values in input-index order (the
// TMA ring); otherwise it is scratch (the direct-load kernel).
template <int THETA, bool RAWCOL, class T>
__device__ __forceinline__ void bulyan_dispatch(T* v, T* col, int stride, int f, const float* const* rowp,
                                                int64_t gidx, float* res) {
  if constexpr (THETA % 2 == 1 && THETA >= 5) {
    if (f == (THETA - 3) / 2) {
      bulyan_column_b3<THETA>(v, RAWCOL ? col : static_cast<const T*>(nullptr), stride, rowp, gidx, res);
      return;
    }
  }
  bulyan_column<THETA>(v, col, stride, f, rowp, gidx, res);
}

// ---------------------------------------------------------------- the kernel
// T = float: thread c of a tile owns coordinate start + c; T = bf2: the two
// coordinates start + 2c, start + 2c + 1.  Either way a tile row is 32 * W
// 32-bit words in shared memory, so the ring geometry is the same and a bf16
// tile covers twice the coordinates for the same bytes.
template <int MODE, int N, int W, class T>
__global__ void __launch_bounds__(32 * (W + kProducers), 1) coord_select_kernel(const __grid_constant__ CoordParams p) {
  constexpr int kConsumerWarps = W;
  constexpr int kTile = 32 * W;                 // T elements per row per tile
  constexpr int EPT = Elem<T>::EPT, ES = Elem<T>::ES;
  constexpr int kCoords = kTile * EPT;          // coordinates per tile
  constexpr int kBulkAlign = 16 / ES;           // coordinates per 16 bytes
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int R = (N > 0) ? N : p.R;
  const int stages = p.stages;
  T* tiles = reinterpret_cast<T*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(stages) * R * kTile * sizeof(T));  // [stages]
  uint64_t* empty = full + stages;
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
      mbar_init(&full[s], kProducers);
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
        const int64_t start = tile * kCoords;
        const int cnt = static_cast<int>((d - start < kCoords ? d - start : int64_t(kCoords)));
        const uint32_t bytes = static_cast<uint32_t>(cnt & ~(kBulkAlign - 1)) * ES;
        uint64_t* bar = &full[stage];
        mbar_arrive_expect_tx(bar, bytes * my_rows);
        if (bytes) {
          T* dst = tiles + size_t(stage) * R * kTile;
          for (int r = q; r < R; r += kProducers) {
            const void* src = reinterpret_cast<const unsigned char*>(rowp[r]) + start * ES;
            if (p.l2_hint) bulk_g2s(dst + r * kTile, src, bytes, bar, pol);
            else bulk_g2s_plain(dst + r * kTile, src, bytes, bar);
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
    mbar_wait(&full[stage], phase);
    const int64_t start = tile * kCoords;
    const int cnt = static_cast<int>((d - start < kCoords ? d - start : int64_t(kCoords)));
    const int bulk_cnt = cnt & ~(kBulkAlign - 1);
    const int c0 = c * EPT;                         // first coordinate of this thread, within the tile
    T* col = tiles + size_t(stage) * R * kTile + c;
    const bool ragged = c0 >= bulk_cnt && c0 < cnt;
    if (ragged) {
      // ragged tail (< 16 bytes per row): not bulk-copied, fetch directly
      for (int r = 0; r < R; ++r) {
        if constexpr (EPT == 1) {
          col[r * kTile] = __ldg(rowp[r] + start + c0);
        } else {
          const unsigned short* rb = reinterpret_cast<const unsigned short*>(rowp[r]);
          const uint32_t lo = __ldg(rb + start + c0);
          const uint32_t hi = (c0 + 1 < cnt) ? __ldg(rb + start + c0 + 1) : 0u;
          col[r * kTile] = T{lo | (hi << 16)};
        }
      }
    }
    if (c0 < cnt) {
      // fused server step: the parameters are loaded before the column work so
      // their latency overlaps it
      float pv[EPT];
#pragma unroll
      for (int h = 0; h < EPT; ++h) pv[h] = (p.extra.sgd && c0 + h < cnt) ? __ldcs(p.out + start + c0 + h) : 0.0f;
      float res[EPT];
      if constexpr (MODE == kModeAverage) {
        avg_column(col, R, kTile, res);
      } else {
        T v[N > 0 ? N : 1];
#pragma unroll
        for (int r = 0; r < N; ++r) v[r] = col[r * kTile];
        if constexpr (MODE == kModeMedian) {
          median_column<N>(v, res);
        } else if constexpr (MODE == kModeTrimmed) {
          trimmed_column<N>(v, p.f, res);
        } else {
          bulyan_dispatch<N, true>(v, col, kTile, p.f, rowp, start + c0, res);
        }
      }
#pragma unroll
      for (int h = 0; h < EPT; ++h)
        if (c0 + h < cnt) store_result(p.out, p.extra, start + c0 + h, res[h], pv[h]);
    }
    // generic-proxy writes into the ring (the ragged-tail fill, Bulyan's sorted
    // column park) must be ordered before the producer's next async-proxy
    // (bulk copy) overwrite of this stage: PTX memory model, ADVICE r1
    if (MODE == kModeBulyan || ragged) fence_proxy_async_smem();
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
        median_column<N>(v, &res);
      } else if constexpr (MODE == kModeTrimmed) {
        trimmed_column<N>(v, p.f, &res);
      } else {
        float* col = reinterpret_cast<float*>(ldg_smem) + threadIdx.x;
        bulyan_dispatch<N, false>(v, col, kLdgThreads, p.f, rowp, k, &res);
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
        median_column<N>(v, &res);
      } else if constexpr (MODE == kModeTrimmed) {
        trimmed_column<N>(v, p.f, &res);
      } else {
        float* col = reinterpret_cast<float*>(ldg_smem) + threadIdx.x;
        bulyan_dispatch<N, false>(v, col, kLdgThreads, p.f, rowp, k, &res);
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
template <int MODE, int N, int W, class T>
inline cudaError_t launch_mode_w(const CoordLaunch& L, cudaStream_t stream) {
  constexpr int kTile = 32 * W;
  constexpr int kCoords = kTile * Elem<T>::EPT;
  constexpr int kThreads = 32 * (W + kProducers);
  CoordParams p;
  for (int i = 0; i < GAR_MAX_N; ++i) p.rows.p[i] = (i < L.n) ? L.rows[i] : nullptr;
  p.idx = L.idx;
  p.out = L.out;
  p.extra = L.extra;
  p.d = L.d;
  p.R = L.R;
  p.f = L.f;
  const size_t stage_bytes = size_t(L.R) * kTile * sizeof(T);
  int stages = static_cast<int>((GAR_RING_KB * 1024) / stage_bytes);
  stages = max(2, min(8, stages));
  p.stages = stages;
  p.l2_hint = l2_evict_first_enabled();
  p.num_tiles = (L.d + kCoords - 1) / kCoords;
  const size_t smem = stages * stage_bytes + 2 * stages * sizeof(uint64_t);
  auto kern = coord_select_kernel<MODE, N, W, T>;
  int occ = 0;
  cudaError_t e = cached_occupancy(kern, kThreads, smem, &occ);
  if (e != cudaSuccess) return e;
  int64_t grid = int64_t(L.num_sms) * occ;
  if (grid > p.num_tiles) grid = p.num_tiles > 0 ? p.num_tiles : 1;
  kern<<<static_cast<unsigned>(grid), kThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

// fp32: the measured loader choice; bf16: always the TMA ring (a bf16 tile
// row carries twice the coordinates of an fp32 one for the same bytes).
template <int MODE, int N, class T>
inline cudaError_t launch_mode(const CoordLaunch& L, cudaStream_t stream) {
  if constexpr (std::is_same<T, float>::value) {
    if (coord_loader_ldg(MODE, L.R)) return launch_ldg<MODE, N>(L, stream);
  }
  if constexpr (N > 0) {
    return launch_mode_w<MODE, N, consumer_warps<MODE, N>(), T>(L, stream);
  } else {
    if (L.R <= 32) return launch_mode_w<MODE, 0, 15, T>(L, stream);
    // above 32 rows: fp32 keeps the measured 7 consumer warps (3 stages);
    // bf16 rows (two coordinates per thread, F2F-heavy sums) take 12 (2 stages
    // of <= 97 KB): C5 sweep, bf16 Average at n = 35: 0.52 ms with 7
    if constexpr (std::is_same<T, float>::value) return launch_mode_w<MODE, 0, 7, T>(L, stream);
    else return launch_mode_w<MODE, 0, 12, T>(L, stream);
  }
}

template <int MODE, int LO, int HI, class T>
inline cudaError_t dispatch_range(const CoordLaunch& L, cudaStream_t stream) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (L.R == LO) return launch_mode<MODE, LO, T>(L, stream);
    return dispatch_range<MODE, LO + 1, HI, T>(L, stream);
  }
}

}  // namespace gar
