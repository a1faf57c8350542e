// mda.cu — MDA selection (§3.3 item 3):
// the subset of q - f inputs with the minimum diameter (largest pairwise
// squared distance, R13), ties to the lexicographically smallest index set,
// on the Gram-derived distance matrix D.  Exhaustive over the C(n, f)
// excluded sets, GPU-parallel:
//   1. mda_prep_kernel (one CTA): the n(n-1)/2 pairs sorted by D descending
//      (rank counting, ties by pair index: deterministic);
//   2. mda_enum_kernel: each thread walks a contiguous run of excluded sets E
//      in lexicographic order (unranked with the combinatorial number system,
//      then advanced in place); the diameter of the kept set is the first pair
//      of the sorted list with neither end in E -- at most f(n-1)+1 probes,
//      usually a handful; per-thread, per-warp and per-CTA minima of
//      (diameter, kept-set order) go to one slot per CTA;
//   3. mda_final_kernel (one CTA): the minimum over the CTA slots, written as
//      the ascending kept indices (the order the average uses, R2).
#include <cstdint>

#include "common.cuh"
#include "gram.h"

namespace gar {

namespace {

constexpr int kMdaThreads = 256;
constexpr int kMaxPairs = GAR_MAX_N * (GAR_MAX_N - 1) / 2;   // 2016

struct Cand {
  double diam;
  uint64_t kept;   // bit i set: input i kept
};

// (diam, kept) order: smaller diameter, then the lexicographically smaller
// sorted index list -- the lowest index where the sets differ belongs to it.
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.diam != b.diam) return a.diam < b.diam;
  const uint64_t x = a.kept ^ b.kept;
  return x != 0 && (a.kept & (x & (~x + 1))) != 0;
}

__global__ void __launch_bounds__(kMdaThreads) mda_prep_kernel(const double* __restrict__ D, int n,
                                                               double* __restrict__ pd, uint16_t* __restrict__ pij) {
  __shared__ double dv[kMaxPairs];
  __shared__ uint16_t iv[kMaxPairs];
  const int P = n * (n - 1) / 2;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    int i = 0, u = p;
    while (u >= n - 1 - i) { u -= n - 1 - i; ++i; }
    const int j = i + 1 + u;
    dv[p] = D[i * n + j];
    iv[p] = static_cast<uint16_t>((i << 8) | j);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const double v = dv[p];
    int rank = 0;
    for (int q = 0; q < P; ++q) rank += (dv[q] > v || (dv[q] == v && q < p)) ? 1 : 0;
    pd[rank] = v;
    pij[rank] = iv[p];
  }
}

__device__ __forceinline__ uint64_t binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  uint64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * static_cast<uint64_t>(n - k + i) / static_cast<uint64_t>(i);
  return r;
}

__global__ void __launch_bounds__(kMdaThreads) mda_enum_kernel(const double* __restrict__ pd,
                                                               const uint16_t* __restrict__ pij, int n, int f,
                                                               uint64_t total, Cand* __restrict__ cta_best) {
  __shared__ double sd[kMaxPairs];
  __shared__ uint16_t sij[kMaxPairs];
  __shared__ Cand warp_best[kMdaThreads / 32];
  const int P = n * (n - 1) / 2;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    sd[p] = pd[p];
    sij[p] = pij[p];
  }
  __syncthreads();
  const uint64_t all = (n == 64) ? ~0ull : ((1ull << n) - 1);
  const uint64_t nthreads = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t per = (total + nthreads - 1) / nthreads;
  const uint64_t r0 = tid * per;
  const uint64_t r1 = (r0 + per < total) ? r0 + per : total;
  Cand best{__longlong_as_double(0x7ff0000000000000ll), 0};
  if (r0 < r1) {
    // unrank r0: the r0-th f-subset of {0..n-1} in lexicographic order
    int e[GAR_MAX_N];
    uint64_t r = r0;
    int x = 0;
    for (int t = 0; t < f; ++t) {
      while (true) {
        const uint64_t c = binom(n - x - 1, f - t - 1);
        if (r < c) break;
        r -= c;
        ++x;
      }
      e[t] = x++;
    }
    uint64_t emask = 0;
    for (int t = 0; t < f; ++t) emask |= 1ull << e[t];
    for (uint64_t rr = r0; rr < r1; ++rr) {
      double diam = 0.0;
      for (int s = 0; s < P; ++s) {
        const int ij = sij[s];
        if (!((emask >> (ij >> 8)) & 1) && !((emask >> (ij & 255)) & 1)) {
          diam = sd[s];
          break;
        }
      }
      const Cand c{diam, all & ~emask};
      if (better(c, best)) best = c;
      // next f-subset in lexicographic order
      int t = f - 1;
      while (t >= 0 && e[t] == n - f + t) --t;
      if (t < 0) break;
      emask &= ~(1ull << e[t]);
      ++e[t];
      emask |= 1ull << e[t];
      for (int u = t + 1; u < f; ++u) {
        emask &= ~(1ull << e[u]);
        e[u] = e[u - 1] + 1;
        emask |= 1ull << e[u];
      }
    }
  }
  // warp, then CTA minimum (fixed shuffle tree: deterministic)
  for (int o = 16; o > 0; o >>= 1) {
    Cand c;
    c.diam = __shfl_xor_sync(0xffffffffu, best.diam, o);
    c.kept = __shfl_xor_sync(0xffffffffu, best.kept, o);
    if (better(c, best)) best = c;
  }
  if ((threadIdx.x & 31) == 0) warp_best[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand b = warp_best[0];
    for (int w = 1; w < kMdaThreads / 32; ++w)
      if (better(warp_best[w], b)) b = warp_best[w];
    cta_best[blockIdx.x] = b;
  }
}

__global__ void mda_final_kernel(const Cand* __restrict__ cta_best, int nb, int n, int32_t* __restrict__ idx_out) {
  if (threadIdx.x != 0) return;
  Cand b = cta_best[0];
  for (int i = 1; i < nb; ++i)
    if (better(cta_best[i], b)) b = cta_best[i];
  int k = 0;
  for (int i = 0; i < n; ++i)
    if ((b.kept >> i) & 1) idx_out[k++] = i;
}

}  // namespace

size_t mda_workspace_bytes(int n) {
  const int P = n * (n - 1) / 2;
  return (size_t(P) * 10 + 15) / 16 * 16 + 16 + size_t(kMdaMaxCtas) * sizeof(Cand);
}

cudaError_t launch_mda_select(const double* D, int n, int f, void* scratch, int num_sms, int32_t* idx_out,
                              cudaStream_t stream) {
  const int P = n * (n - 1) / 2;
  double* pd = reinterpret_cast<double*>(scratch);
  uint16_t* pij = reinterpret_cast<uint16_t*>(pd + (P > 0 ? P : 1));
  Cand* cta = reinterpret_cast<Cand*>(reinterpret_cast<unsigned char*>(scratch) +
                                      ((size_t(P) * 10 + 15) / 16 * 16 + 16));
  uint64_t total = 1;
  for (int i = 1; i <= f; ++i) total = total * uint64_t(n - f + i) / uint64_t(i);
  int blocks = num_sms * 4;
  if (blocks > kMdaMaxCtas) blocks = kMdaMaxCtas;
  const uint64_t need = (total + kMdaThreads - 1) / kMdaThreads;
  if (need < uint64_t(blocks)) blocks = static_cast<int>(need > 0 ? need : 1);
  if (P > 0) mda_prep_kernel<<<1, kMdaThreads, 0, stream>>>(D, n, pd, pij);
  mda_enum_kernel<<<blocks, kMdaThreads, 0, stream>>>(pd, pij, n, f, total, cta);
  mda_final_kernel<<<1, 32, 0, stream>>>(cta, blocks, n, idx_out);
  return cudaGetLastError();
}

}  // namespace gar
