// exchange.cu — the d-sharded Krum-family exchange (row a10, PAPER.md
// l.437-438) fused into peer-memory kernels instead of an NCCL all-reduce:
// every rank reduces its per-CTA partial Gram matrices, stores the result
// into its own slot of EVERY rank's slot array (NVLink peer stores into
// symmetric memory), signals each rank's flag with a system-scope release,
// waits (acquire) until all ranks' flags carry this call's epoch, and sums
// the world slots in rank order.  Every rank therefore holds the bit-identical
// whole-vector Gram matrix, and no collective library call sits on the path.
#include <cstdint>

#include "common.cuh"
#include "gram.h"

namespace gar {

namespace {

// G_local = sum of the CTA partials (same order as gram_reduce_kernel: one
// warp per entry, lane-strided sums, xor-shuffle tree), stored at slot `rank`
// of every rank's slot array.
__global__ void __launch_bounds__(256) gram_reduce_bcast_kernel(const double* __restrict__ partials, int n_parts,
                                                                int nn, PeerSlots slots, int world, int rank) {
  const int e = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= nn) return;
  double s = 0.0;
  for (int p = lane; p < n_parts; p += 32) s += partials[static_cast<size_t>(p) * nn + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane < world) slots.p[lane][static_cast<size_t>(rank) * nn + e] = s;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Block 0 publishes this rank's slot writes (they completed with the previous
// kernel) to every rank's flag[rank]; every block then waits until all
// `world` local flags reach `epoch` and sums the slots in rank order.  A wait
// longer than ~10 s (a rank that never arrives) traps: the kernel fails, the
// stream (and context) carry a sticky launch error that the next libgar /
// CUDA call returns (GAR_ERR_CUDA), instead of hanging the GPU or handing a
// plausible-looking selection to the caller.
__global__ void __launch_bounds__(256) gram_gather_kernel(PeerFlags flags, int world, int rank, uint32_t epoch,
                                                          const double* __restrict__ local_slots, int nn,
                                                          double* __restrict__ G) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_system();
    for (int r = 0; r < world; ++r) st_release_sys(flags.p[r] + rank, epoch);
  }
  if (threadIdx.x == 0) {
    const uint32_t* mine = flags.p[rank];
    const uint64_t t0 = global_ns();
    for (int r = 0; r < world; ++r) {
      while (static_cast<int32_t>(ld_acquire_sys(mine + r) - epoch) < 0) {
        if (global_ns() - t0 > 10000000000ull) __trap();
        __nanosleep(100);
      }
    }
  }
  __syncthreads();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nn) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += local_slots[static_cast<size_t>(r) * nn + e];
  G[e] = s;
}

}  // namespace

cudaError_t launch_gram_exchange(const double* partials, int n_parts, int n, const PeerSlots& slots,
                                 const PeerFlags& flags, int world, int rank, uint32_t epoch, double* G,
                                 cudaStream_t stream) {
  const int nn = n * n;
  gram_reduce_bcast_kernel<<<(nn + 7) / 8, 256, 0, stream>>>(partials, n_parts, nn, slots, world, rank);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  gram_gather_kernel<<<(nn + 255) / 256, 256, 0, stream>>>(flags, world, rank, epoch, slots.p[rank], nn, G);
  return cudaGetLastError();
}

}  // namespace gar
