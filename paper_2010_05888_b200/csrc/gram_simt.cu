// gram_simt.cu — CUDA-core Gram partials with fp64 products (reference-quality
// cross-check for the tensor-core Gram kernel; not on the product path once
// gram_tc.cu is in place), plus the deterministic partial reduction.
#include <cmath>

#include "common.cuh"
#include "gram.h"

namespace gar {

namespace {

constexpr int kSimtThreads = 256;
constexpr int kSimtTile = 64;

__device__ __forceinline__ float fin(float v) { return isfinite(v) ? v : 0.0f; }

__device__ __forceinline__ float med3(float a, float b, float c) {
  return fmaxf(fminf(a, b), fminf(fmaxf(a, b), c));
}

__global__ void __launch_bounds__(kSimtThreads) gram_simt_kernel(const __grid_constant__ RowPtrs rows, int n,
                                                                 int64_t d, int64_t chunk,
                                                                 double* partials) {
  __shared__ float h[GAR_MAX_N][kSimtTile + 1];
  __shared__ float cref[kSimtTile];
  const int npairs = n * (n + 1) / 2;
  double acc[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  int pi[9], pj[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    int p = threadIdx.x + q * kSimtThreads, i = 0;
    if (p < npairs) {
      while (p >= n - i) { p -= n - i; ++i; }
      pi[q] = i;
      pj[q] = i + p;
    } else {
      pi[q] = pj[q] = -1;
    }
  }
  const int64_t lo = blockIdx.x * chunk;
  const int64_t hi = (d < lo + chunk) ? d : lo + chunk;
  for (int64_t k0 = lo; k0 < hi; k0 += kSimtTile) {
    const int cnt = static_cast<int>(hi - k0 < kSimtTile ? hi - k0 : kSimtTile);
    if (threadIdx.x < kSimtTile) {
      float c = 0.0f;
      if (threadIdx.x < cnt) {
        const int64_t k = k0 + threadIdx.x;
        c = fin(rows.p[0][k]);
        if (n >= 3) c = med3(c, fin(rows.p[1][k]), fin(rows.p[2][k]));
      }
      cref[threadIdx.x] = c;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * kSimtTile; e += kSimtThreads) {
      const int i = e / kSimtTile, k = e % kSimtTile;
      h[i][k] = (k < cnt) ? __fsub_rn(rows.p[i][k0 + k], cref[k]) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      if (pi[q] >= 0) {
        const float* a = h[pi[q]];
        const float* b = h[pj[q]];
        double s = acc[q];
        for (int k = 0; k < kSimtTile; ++k) s = fma(static_cast<double>(a[k]), static_cast<double>(b[k]), s);
        acc[q] = s;
      }
    }
    __syncthreads();
  }
  double* P = partials + static_cast<size_t>(blockIdx.x) * n * n;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if (pi[q] >= 0) {
      P[pi[q] * n + pj[q]] = acc[q];
      P[pj[q] * n + pi[q]] = acc[q];
    }
  }
}

// 256 threads = 32 entries x 8 partial groups; fixed-order sums.
// One warp per Gram entry: lane l sums partials l, l+32, ... (independent
// loads in flight together), then a fixed xor-shuffle tree -- a deterministic
// order, and latency ~ one memory round trip instead of n_parts/8 dependent ones.
__global__ void __launch_bounds__(256) gram_reduce_kernel(const double* __restrict__ partials, int n_parts,
                                                          int nn, double* __restrict__ G) {
  const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= nn) return;
  double s = 0.0;
  for (int p = lane; p < n_parts; p += 32) s += partials[static_cast<size_t>(p) * nn + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) G[e] = s;
}

}  // namespace

cudaError_t launch_gram_partials_simt(const float* const* rows, int n, int64_t d, double* partials,
                                      int num_sms, int* n_parts, cudaStream_t stream) {
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  int parts = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  int64_t chunk = (d + parts - 1) / parts;
  chunk = (chunk + kSimtTile - 1) / kSimtTile * kSimtTile;
  if (chunk < kSimtTile) chunk = kSimtTile;
  parts = static_cast<int>((d + chunk - 1) / chunk);
  if (parts < 1) parts = 1;
  gram_simt_kernel<<<parts, kSimtThreads, 0, stream>>>(rp, n, d, chunk, partials);
  *n_parts = parts;
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const double* partials, int n_parts, int n, double* G, cudaStream_t stream) {
  const int nn = n * n;
  gram_reduce_kernel<<<(nn + 7) / 8, 256, 0, stream>>>(partials, n_parts, nn, G);
  return cudaGetLastError();
}

}  // namespace gar
