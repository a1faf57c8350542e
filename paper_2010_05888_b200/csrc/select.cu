// select.cu — from the summed Gram matrix to the Krum / Multi-Krum / Bulyan
// selection (rows a5 epilogue, a6, a7 of DESIGN.md §1) as its own launch: one
// CTA of 256 threads runs sel::select_block (select_block.cuh; the n x n
// problem, n <= 64, lives in shared memory).
#include "select_block.cuh"

namespace gar {

namespace {

constexpr int kSelThreads = 256;

__global__ void __launch_bounds__(kSelThreads) select_kernel(const double* __restrict__ G, int n, int f, int m,
                                                             int rule, int32_t* __restrict__ idx_out,
                                                             double* __restrict__ D_out) {
  extern __shared__ __align__(16) unsigned char sel_smem[];
  sel::select_block(G, n, f, m, rule, idx_out, D_out, *reinterpret_cast<sel::SelSmem*>(sel_smem), threadIdx.x,
                    kSelThreads, 1);
}

}  // namespace

cudaError_t launch_select(const double* G, int n, int f, int m, int rule, int32_t* idx_out, double* D_out,
                          cudaStream_t stream) {
  int occ = 0;
  cudaError_t e = cached_occupancy(select_kernel, kSelThreads, sizeof(sel::SelSmem), &occ);
  if (e != cudaSuccess) return e;
  select_kernel<<<1, kSelThreads, sizeof(sel::SelSmem), stream>>>(G, n, f, m, rule, idx_out, D_out);
  return cudaGetLastError();
}

}  // namespace gar
