// membership.cu — trimmed-set membership (verification entry point,
// gar_trimmed_membership): per coordinate, bit i of mask[k] is set iff input i
// is among the n - 2f values the trimmed mean keeps (row a3; the north_star's
// bit-exact "trimmed-set membership").  The product trimmed mean runs a
// data-oblivious network that never tracks indices; this kernel states the
// membership explicitly by rank counting over (canonical value, index)
// (R1, R5): kept_i  <=>  f <= #{j : (c_j, j) < (c_i, i)} < n - f.
// O(n^2) per coordinate: a checking path, not a hot one.
#include <cstdint>

#include "common.cuh"

namespace gar {

namespace {

__global__ void __launch_bounds__(256) trimmed_membership_kernel(const __grid_constant__ RowPtrs rows, int n,
                                                                 int f, int64_t d, uint64_t* __restrict__ mask) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < d; k += int64_t(gridDim.x) * blockDim.x) {
    float c[GAR_MAX_N];
#pragma unroll 8
    for (int i = 0; i < n; ++i) c[i] = canon(__ldg(rows.p[i] + k));
    uint64_t m = 0;
    for (int i = 0; i < n; ++i) {
      int rank = 0;
      for (int j = 0; j < n; ++j) rank += (c[j] < c[i] || (c[j] == c[i] && j < i)) ? 1 : 0;
      if (rank >= f && rank < n - f) m |= uint64_t(1) << i;
    }
    mask[k] = m;
  }
}

// Rows holding any non-finite value (SPEC's vector-level sanitize):
// blockIdx.y = row, grid-stride float4 chunks, one warp vote and at most one
// atomicOr per warp.  Reads every input byte once (HBM-bound).
__global__ void __launch_bounds__(256) nonfinite_rows_kernel(const __grid_constant__ RowPtrs rows, int64_t d,
                                                             unsigned long long* __restrict__ mask) {
  const int r = blockIdx.y;
  const float* row = rows.p[r];
  bool bad = false;
  const int64_t n4 = d >> 2;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n4; q += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(row) + q);
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
  }
  const int64_t k = (n4 << 2) + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (blockIdx.x == 0 && k < d) bad |= !isfinite(row[k]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(mask, 1ull << r);
}

}  // namespace

cudaError_t launch_nonfinite_rows(const float* const* rows, int n, int64_t d, uint64_t* mask, int num_sms,
                                  cudaStream_t stream) {
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  cudaError_t e = cudaMemsetAsync(mask, 0, sizeof(uint64_t), stream);
  if (e != cudaSuccess) return e;
  int64_t bx = (d / 4 + 255) / 256;
  const int64_t cap = (int64_t(num_sms) * 8 + n - 1) / n;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  nonfinite_rows_kernel<<<dim3(static_cast<unsigned>(bx), n), 256, 0, stream>>>(
      rp, d, reinterpret_cast<unsigned long long*>(mask));
  return cudaGetLastError();
}

cudaError_t launch_trimmed_membership(const float* const* rows, int n, int f, int64_t d, uint64_t* mask,
                                      int num_sms, cudaStream_t stream) {
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  int64_t blocks = (d + 255) / 256;
  const int64_t cap = int64_t(num_sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  trimmed_membership_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(rp, n, f, d, mask);
  return cudaGetLastError();
}

}  // namespace gar
