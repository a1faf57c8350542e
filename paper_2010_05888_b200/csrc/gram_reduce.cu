// gram_reduce.cu — the deterministic reduction of the Gram kernel's per-CTA
// partial matrices (row a5): G = sum of the partials in a fixed order.
#include "common.cuh"
#include "gram.h"

namespace gar {

namespace {

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

cudaError_t launch_gram_reduce(const double* partials, int n_parts, int n, double* G, cudaStream_t stream) {
  const int nn = n * n;
  gram_reduce_kernel<<<(nn + 7) / 8, 256, 0, stream>>>(partials, n_parts, nn, G);
  return cudaGetLastError();
}

}  // namespace gar
