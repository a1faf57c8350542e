// select_block.cuh — the Krum / Multi-Krum / Bulyan selection from the summed
// Gram matrix, as a block-level device function (rows a5 epilogue, a6, a7 of
// DESIGN.md §1).  Run by `nthreads` threads of one CTA (>= 64, synchronised on
// named barrier `bar`) over the SelSmem scratch; select_kernel (select.cu)
// runs it with 256 threads.
//
//   D_ij = G_ii + G_jj - 2 G_ij   (fp64, evaluated once per unordered pair so D
//          is bitwise symmetric; < 0 -> 0; non-finite or > FLT_MAX -> +inf, R4)
//   row i sorted ascending by (D_ij, j) via rank counting (n^3 independent
//   compares spread over the threads)
//   Krum score s_i = sum of the k smallest D_ij, j in pool, j != i, in ascending
//   order (fp64), k = n-f-2 (Multi-Krum) or max(|R|-f-2, 0) (Bulyan round, R7)
//   Multi-Krum: the m smallest (s_i, i);  Bulyan: theta = n-2f rounds of
//   argmin (s_i, i) with removal, on the same cached D.
#pragma once
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "gram.h"
#include "gram_common.cuh"

namespace gar {
namespace sel {

struct SelSmem {
  double Dm[GAR_MAX_N][GAR_MAX_N + 1];
  double sd[GAR_MAX_N][GAR_MAX_N];          // row i ascending, j != i
  unsigned char sj[GAR_MAX_N][GAR_MAX_N];
  double score[GAR_MAX_N];
  double wbest[2][2];                       // Bulyan rounds, n > 32: the two warps' winners
  int wbi[2][2];
  unsigned long long pool;
};

__device__ __forceinline__ bool key_lt(double a, int ia, double b, int ib) {
  return a < b || (a == b && ia < ib);
}

// Bulyan's theta rounds on W warps: thread i < n holds row i's distances in
// ascending order (ROWS >= n - 1 registers) and their column indices; per
// round, its score over the pool, then the argmin of (score, index): a warp
// shuffle tree, and for W = 2 the two warp winners through shared memory
// (one named barrier `bar2` of 64 threads per round, slots alternating).
template <int ROWS, int W>
__device__ __forceinline__ void bulyan_rounds(SelSmem& S, int n, int f, int theta, int32_t* __restrict__ idx_out,
                                              int tid, int bar2) {
  const int i = tid, lane = tid & 31, warp = tid >> 5;
  double row[ROWS];
  uint32_t rj4[(ROWS + 3) / 4];                    // column indices, 4 bytes per register
#pragma unroll
  for (int q = 0; q < (ROWS + 3) / 4; ++q) rj4[q] = 0;
#pragma unroll
  for (int e = 0; e < ROWS; ++e) {
    const bool ok = i < n && e < n - 1;
    row[e] = ok ? S.sd[i][e] : 0.0;
    rj4[e >> 2] |= static_cast<uint32_t>(ok ? S.sj[i][e] : 0) << (8 * (e & 3));
  }
  unsigned long long P = (n == 64) ? ~0ull : ((1ull << n) - 1ull);
  for (int t = 0; t < theta; ++t) {
    const int k = max(__popcll(P) - f - 2, 0);
    double sc = 0.0;
    int taken = 0;
#pragma unroll
    for (int e = 0; e < ROWS; ++e) {
      const int j = (rj4[e >> 2] >> (8 * (e & 3))) & 0xFF;
      const bool take = e < n - 1 && ((P >> j) & 1ull) && taken < k;
      if (take) sc += row[e];
      taken += take ? 1 : 0;
    }
    const bool in = i < n && ((P >> i) & 1ull);
    double best = in ? sc : INFINITY;
    int bi = in ? i : (1 << 30);
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (key_lt(ob, oi, best, bi)) {
        best = ob;
        bi = oi;
      }
    }
    if constexpr (W == 2) {
      const int slot = t & 1;
      if (lane == 0) {
        S.wbest[slot][warp] = best;
        S.wbi[slot][warp] = bi;
      }
      gram::named_bar(bar2, 64);
      const double b0 = S.wbest[slot][0], b1 = S.wbest[slot][1];
      const int i0 = S.wbi[slot][0], i1 = S.wbi[slot][1];
      bi = key_lt(b1, i1, b0, i0) ? i1 : i0;
    }
    if (i == 0) idx_out[t] = bi;
    P &= ~(1ull << bi);
  }
}

__device__ __forceinline__ void select_block(const double* __restrict__ G, int n, int f, int m, int rule,
                                             int32_t* __restrict__ idx_out, double* __restrict__ D_out,
                                             SelSmem& S, int tid, int nthreads, int bar) {
  using gram::named_bar;
  auto& Dm = S.Dm;
  auto& sd = S.sd;
  auto& sj = S.sj;
  auto& score = S.score;
  auto& pool = S.pool;
  for (int e = tid; e < n * n; e += nthreads) {
    const int i = e / n, j = e % n;
    double v = 0.0;
    if (i != j) {
      const int a = min(i, j), b = max(i, j);
      v = G[a * n + a] + G[b * n + b] - 2.0 * G[a * n + b];
      if (!(v >= 0.0)) v = (v < 0.0) ? 0.0 : INFINITY;   // NaN -> +inf, negative -> 0
      if (v > static_cast<double>(FLT_MAX)) v = INFINITY;
    }
    Dm[i][j] = v;
    if (D_out) D_out[e] = v;
  }
  named_bar(bar, nthreads);
  if (rule == kSelDistancesOnly) return;

  // rank of (D_ij, j) within row i (j != i) -> position in the sorted row
  for (int e = tid; e < n * n; e += nthreads) {
    const int i = e / n, j = e % n;
    if (i == j) continue;
    const double v = Dm[i][j];
    int r = 0;
    for (int k = 0; k < n; ++k)
      if (k != i && key_lt(Dm[i][k], k, v, j)) ++r;
    sd[i][r] = v;
    sj[i][r] = static_cast<unsigned char>(j);
  }
  if (tid == 0) pool = (n == 64) ? ~0ull : ((1ull << n) - 1ull);
  named_bar(bar, nthreads);

  if (rule == kSelMultiKrum) {
    const int k = n - f - 2;
    if (tid < n) {
      double s = 0.0;
      for (int r = 0; r < k; ++r) s += sd[tid][r];
      score[tid] = s;
    }
    named_bar(bar, nthreads);
    if (tid < n) {
      int r = 0;
      for (int j = 0; j < n; ++j)
        if (key_lt(score[j], j, score[tid], tid)) ++r;
      if (r < m) idx_out[r] = tid;
    }
    return;
  }

  const int theta = n - 2 * f;
  // Bulyan: theta rounds of Krum with removal (R7).  Thread i (one warp for
  // n <= 32, two for n <= 64) holds row i's sorted distances in registers;
  // each round sums the k smallest pool members in ascending order (fp64, the
  // oracle's additions) and an argmin over (score, index) picks the next.
  if (n <= 32) {
    if (tid < 32) bulyan_rounds<31, 1>(S, n, f, theta, idx_out, tid, bar + 1);
  } else {
    if (tid < 64) bulyan_rounds<63, 2>(S, n, f, theta, idx_out, tid, bar + 1);
  }
}

}  // namespace sel
}  // namespace gar
