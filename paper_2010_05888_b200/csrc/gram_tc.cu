// gram_tc.cu — the pairwise-distance contraction on the 5th-gen tensor cores
// (row a5 of DESIGN.md §1): per-CTA partial Gram matrices of the centred rows,
//     G_ij = sum_k (x_ik - c_k)(x_jk - c_k),
// from which select.cu forms D_ij = G_ii + G_jj - 2 G_ij ("norm correction").
//
// Precision: h = x - c is split as h = hi + lo with
// hi = rna_tf32(h) and lo = rna_tf32(h - hi); one tcgen05.mma kind::tf32 per
// K-step multiplies A = [H; L] (M = 2*NP rows) by B = H (N = NP rows):
//     D = [H H^T ; L H^T]   ->   G = H H^T + L H^T + (L H^T)^T
// (3 of the 4 split products; the dropped lo*lo is < 2^-22 relative).  TMEM
// fp32 accumulators are drained every KT coordinates into fp64 registers.
//
// Warp roles (one persistent CTA per SM):
//   7-8 warps   loaders: LDG.128 (streaming, evict-first) with a P-deep register
//               prefetch ring, centring, hi/lo split, STS into the SWIZZLE_128B
//               K-major operand layout, fence.proxy.async, mbarrier arrive;
//   4 or 8 warps epilogue: tcgen05.ld of the accumulator lanes -> fp64 sums
//               (8 when NP = 64: each thread owns half of a 64-column row);
//   last warp   TMEM allocator + single-thread tcgen05.mma issuer.
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "gram.h"

namespace gar {

namespace {

template <int NP_>
struct Cfg {
  static constexpr int NP = NP_;                 // padded row count (32 or 64)
  static constexpr int M = 2 * NP;               // MMA M: H rows then L rows
  static constexpr int N = NP;                   // MMA N: H rows
  static constexpr int KT = 128;                 // coordinates per stage (tile)
  static constexpr int ATOMS = KT / 32;          // 128-byte K atoms per stage
  static constexpr int ATOM_BYTES = M * 128;     // one K atom of A (8-row groups of 1 KB)
  static constexpr int STAGE_BYTES = ATOMS * ATOM_BYTES;
  static constexpr int STAGES = (NP == 32) ? 4 : 3;
  // Register budget: the CTA's warp count is rounded up to a multiple of 4 for
  // register allocation, so 13 warps (NP = 32) and 16 warps (NP = 64) both
  // leave 128 registers per thread.
  static constexpr int LOADER_WARPS = (NP == 32) ? 8 : 7;
  static constexpr int RPW = (NP + LOADER_WARPS - 1) / LOADER_WARPS;  // rows per loader warp (4 / 10)
  static constexpr int PREFETCH = (NP == 32) ? 3 : 2;
  static constexpr int EPI_WARP0 = LOADER_WARPS;
  static constexpr int EPI_WARPS = (NP == 32) ? 4 : 8;    // 4 sub-partitions x column halves
  static constexpr int EPI_COLS = N / (EPI_WARPS / 4);    // accumulator columns per epilogue thread
  static constexpr int MMA_WARP = EPI_WARP0 + EPI_WARPS;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr int TMEM_COLS = 2 * N;        // double-buffered accumulator
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * KT * 4 /*c_buf*/ +
                                    (2 * STAGES + 4) * 8 /*barriers*/ + 16;
  static_assert(KT / 4 == 32, "one float4 chunk per lane per row");
};

// ---- tcgen05 / descriptor helpers ------------------------------------------
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
  // SM100 shared-memory matrix descriptor, K-major, SWIZZLE_128B:
  // start>>4 [0,14), LBO>>4 [16,30) (unused for swizzled K-major: 1), SBO>>4
  // [32,46) = 1024 B between 8-row groups, version [46,48) = 1, layout [61,64) = 2.
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

template <int M, int N>
__host__ __device__ constexpr uint32_t tf32_idesc() {
  // kind::tf32 instruction descriptor: D fp32 [4,6)=1, A tf32 [7,10)=2,
  // B tf32 [10,13)=2, both K-major, N>>3 at [17,23), M>>4 at [24,29).
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
        "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ float fin(float v) { return isfinite(v) ? v : 0.0f; }

__device__ __forceinline__ float med3(float a, float b, float c) {
  return fmaxf(fminf(a, b), fminf(fmaxf(a, b), c));
}

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ float4 load_chunk(const float* row, int64_t k0, int64_t d) {
  if (k0 + 4 <= d) return __ldcs(reinterpret_cast<const float4*>(row + k0));
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k0 + 0 < d) v.x = __ldcs(row + k0 + 0);
  if (k0 + 1 < d) v.y = __ldcs(row + k0 + 1);
  if (k0 + 2 < d) v.z = __ldcs(row + k0 + 2);
  return v;
}

// Byte offset of (row, 16-byte chunk c16 within a K atom) in the SW128 K-major layout.
__device__ __forceinline__ uint32_t sw128_offset(int row, int c16) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((c16 ^ (row & 7)) << 4));
}

// Centre-row pick (runs on all threads of the CTA, uses `scratch` shared memory,
// leaves the chosen row index in scratch[0] as an int).  Deterministic.
template <class C>
__device__ void center_pick(const RowPtrs& rows, int n, int64_t d, int64_t k_begin, unsigned char* scratch) {
  constexpr int S = 256;                                   // sample coordinates
  float* xs = reinterpret_cast<float*>(scratch);           // [n][S]
  float* Ds = xs + GAR_MAX_N * S;                          // [64][65]
  float* score = Ds + GAR_MAX_N * (GAR_MAX_N + 1);         // [64]
  if (n <= 2) {
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<int*>(scratch) = 0;
    __syncthreads();
    return;
  }
  for (int e = threadIdx.x; e < n * (S / 4); e += C::THREADS) {
    const int r = e / (S / 4), q = e % (S / 4);
    const float4 v = load_chunk(rows.p[r], k_begin + 4 * q, d);
    reinterpret_cast<float4*>(xs + r * S)[q] = make_float4(fin(v.x), fin(v.y), fin(v.z), fin(v.w));
  }
  __syncthreads();
  const int np = n * (n - 1) / 2;
  for (int p = threadIdx.x; p < np; p += C::THREADS) {
    int i = 0, t = p;
    while (t >= n - 1 - i) { t -= n - 1 - i; ++i; }
    const int j = i + 1 + t;
    const float4* a = reinterpret_cast<const float4*>(xs + i * S);
    const float4* b = reinterpret_cast<const float4*>(xs + j * S);
    float acc = 0.f;
    for (int k = 0; k < S / 4; ++k) {
      const float4 u = a[k], v = b[k];
      const float dx = u.x - v.x, dy = u.y - v.y, dz = u.z - v.z, dw = u.w - v.w;
      acc = fmaf(dx, dx, acc); acc = fmaf(dy, dy, acc); acc = fmaf(dz, dz, acc); acc = fmaf(dw, dw, acc);
    }
    if (!(acc <= 3.0e38f)) acc = __int_as_float(0x7f800000);
    Ds[i * (GAR_MAX_N + 1) + j] = acc;
    Ds[j * (GAR_MAX_N + 1) + i] = acc;
  }
  __syncthreads();
  const int h = (n - 1) / 2;
  if (threadIdx.x < n) {
    const int i = threadIdx.x;
    // sum of the h smallest D_ij (j != i), ties by index, ascending order
    float s = 0.f;
    int last_j = -1;
    float last_v = -1.f;
    for (int t = 0; t < h; ++t) {
      float bv = __int_as_float(0x7f800000);
      int bj = -1;
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        const float v = Ds[i * (GAR_MAX_N + 1) + j];
        const bool after = (v > last_v) || (v == last_v && j > last_j);
        if (after && (bj < 0 || v < bv || (v == bv && j < bj))) { bv = v; bj = j; }
      }
      s += bv;
      last_v = bv;
      last_j = bj;
    }
    score[i] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int best = 0;
    for (int i = 1; i < n; ++i)
      if (score[i] < score[best]) best = i;
    *reinterpret_cast<int*>(scratch) = best;
  }
  __syncthreads();
}

template <int NP>
__global__ void __launch_bounds__(Cfg<NP>::THREADS, 1)
    gram_tc_kernel(const __grid_constant__ RowPtrs rows, int n, int64_t d, int64_t num_tiles,
                   double* __restrict__ partials) {
  using C = Cfg<NP>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* stages = base;
  float4* c_buf = reinterpret_cast<float4*>(base + C::STAGES * C::STAGE_BYTES);   // [2][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::STAGES * C::STAGE_BYTES + 2 * C::KT * 4);
  uint64_t* stage_free = full + C::STAGES;
  uint64_t* acc_full = stage_free + C::STAGES;     // [2]
  uint64_t* acc_empty = acc_full + 2;              // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  // contiguous, balanced tile range [t0, t0 + T) of this CTA
  const int64_t t0 = num_tiles * blockIdx.x / G;
  const int64_t T = num_tiles * (blockIdx.x + 1) / G - t0;

  // ---- centring row r* of this CTA: the most central row of a
  // 256-coordinate sample of the CTA's own slice, score_i = sum of the
  // floor((n-1)/2) smallest sample distances D_ij (a Krum score with the
  // largest f any rule admits).  Per-coordinate centring is a translation, so
  // each CTA may pick its own row.
  __shared__ int center_row;
  center_pick<C>(rows, n, d, t0 * C::KT, stages);
  if (threadIdx.x == 0) center_row = *reinterpret_cast<int*>(stages);
  __syncthreads();
  const int rc = center_row;
  // zero the operand ring once: rows >= n are never written afterwards
  for (int i = threadIdx.x; i < C::STAGES * C::STAGE_BYTES / 16; i += C::THREADS)
    reinterpret_cast<float4*>(stages)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], C::LOADER_WARPS);
      mbar_init(&stage_free[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], C::EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < C::LOADER_WARPS) {
    // ====================================================== loaders
    const int q = lane;                         // float4 chunk of the tile (coords 4q..4q+3)
    const int atom = q >> 3, c16 = q & 7;
    float4 ring[C::PREFETCH][C::RPW + 1];          // + the centre row (warp 0 only)
    const float* crow = rows.p[rc];
#pragma unroll
    for (int p = 0; p < C::PREFETCH; ++p) {
      const int64_t k0 = (t0 + p) * C::KT + 4 * q;
#pragma unroll
      for (int j = 0; j < C::RPW; ++j) {
        const int r = warp * C::RPW + j;
        ring[p][j] = (p < T && r < n) ? load_chunk(rows.p[r], k0, d) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      ring[p][C::RPW] = (p < T && warp == 0) ? load_chunk(crow, k0, d) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i0 = 0; i0 < T; i0 += C::PREFETCH) {
#pragma unroll
      for (int p = 0; p < C::PREFETCH; ++p) {
        const int64_t i = i0 + p;
        if (i >= T) break;
        const int s = static_cast<int>(i % C::STAGES);
        const uint32_t use = static_cast<uint32_t>(i / C::STAGES);
        float4* x = ring[p];
        // centring reference c_k = fin(x_{r*,k})
        float4* cb = c_buf + (i & 1) * 32;
        if (warp == 0) {
          const float4 xc = x[C::RPW];
          cb[q] = make_float4(fin(xc.x), fin(xc.y), fin(xc.z), fin(xc.w));
        }
        named_bar(1, C::LOADER_WARPS * 32);
        const float4 c = cb[q];
        if (use > 0) mbar_wait(&stage_free[s], (use - 1) & 1);
        unsigned char* A = stages + s * C::STAGE_BYTES + atom * C::ATOM_BYTES;
#pragma unroll
        for (int j = 0; j < C::RPW; ++j) {
          const int r = warp * C::RPW + j;
          if (r < n) {
            float4 h, hi, lo;
            h.x = __fsub_rn(x[j].x, c.x); h.y = __fsub_rn(x[j].y, c.y);
            h.z = __fsub_rn(x[j].z, c.z); h.w = __fsub_rn(x[j].w, c.w);
            hi.x = rna_tf32(h.x); hi.y = rna_tf32(h.y); hi.z = rna_tf32(h.z); hi.w = rna_tf32(h.w);
            lo.x = rna_tf32(__fsub_rn(h.x, hi.x)); lo.y = rna_tf32(__fsub_rn(h.y, hi.y));
            lo.z = rna_tf32(__fsub_rn(h.z, hi.z)); lo.w = rna_tf32(__fsub_rn(h.w, hi.w));
            *reinterpret_cast<float4*>(A + sw128_offset(r, c16)) = hi;
            *reinterpret_cast<float4*>(A + sw128_offset(NP + r, c16)) = lo;
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        // refill this ring slot with tile i + PREFETCH
        const int64_t k0 = (t0 + i + C::PREFETCH) * C::KT + 4 * q;
        const bool more = i + C::PREFETCH < T;
#pragma unroll
        for (int j = 0; j < C::RPW; ++j) {
          const int r = warp * C::RPW + j;
          if (more && r < n) x[j] = load_chunk(rows.p[r], k0, d);
        }
        if (more && warp == 0) x[C::RPW] = load_chunk(crow, k0, d);
      }
    }
  } else if (warp == C::MMA_WARP) {
    // ====================================================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc<C::M, C::N>();
      const uint32_t stage0 = smem_u32(stages);
      for (int64_t i = 0; i < T; ++i) {
        const int s = static_cast<int>(i % C::STAGES);
        const int buf = static_cast<int>(i & 1);
        const uint32_t nb = static_cast<uint32_t>(i >> 1);
        if (nb > 0) mbar_wait(&acc_empty[buf], (nb - 1) & 1);
        mbar_wait(&full[s], static_cast<uint32_t>(i / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * C::N;
#pragma unroll
        for (int kk = 0; kk < C::KT / 8; ++kk) {
          const uint32_t a = stage0 + s * C::STAGE_BYTES + (kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32;
          const uint64_t desc = sw128_desc(a);
          mma_tf32(d_tmem, desc, desc, idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&stage_free[s]);
        mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ====================================================== epilogue (TMEM -> fp64)
    const int ew = warp - C::EPI_WARP0;
    const int e = warp & 3;                      // TMEM sub-partition of this warp
    const int col0 = (ew >> 2) * C::EPI_COLS;    // column half (NP = 64) or 0
    double acc[C::EPI_COLS];
#pragma unroll
    for (int j = 0; j < C::EPI_COLS; ++j) acc[j] = 0.0;
    for (int64_t i = 0; i < T; ++i) {
      const int buf = static_cast<int>(i & 1);
      mbar_wait(&acc_full[buf], static_cast<uint32_t>(i >> 1) & 1);
      tc_fence_after();
      float v[C::EPI_COLS];
#pragma unroll
      for (int h = 0; h < C::EPI_COLS / 32; ++h)
        tmem_ld32(tmem_base + (static_cast<uint32_t>(32 * e) << 16) + buf * C::N + col0 + 32 * h, v + 32 * h);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
#pragma unroll
      for (int j = 0; j < C::EPI_COLS; ++j) acc[j] += static_cast<double>(v[j]);
    }
    // D row held by this thread: M=64 -> lanes 0-15 of each sub-partition; M=128 -> all lanes
    int m = -1;
    if (C::M == 64) {
      if (lane < 16) m = 16 * e + lane;
    } else {
      m = 32 * e + lane;
    }
    // park T = H H^T (rows 0..NP-1) and B = L H^T (rows NP..2NP-1) in shared memory
    constexpr int EPI_THREADS = C::EPI_WARPS * 32;
    double* TB = reinterpret_cast<double*>(stages);       // [2NP][NP+1]; operand ring is idle now
    named_bar(2, EPI_THREADS);
    if (m >= 0) {
#pragma unroll
      for (int j = 0; j < C::EPI_COLS; ++j) TB[m * (NP + 1) + col0 + j] = acc[j];
    }
    named_bar(2, EPI_THREADS);
    double* P = partials + static_cast<size_t>(blockIdx.x) * n * n;
    for (int idx = threadIdx.x - C::EPI_WARP0 * 32; idx < n * n; idx += EPI_THREADS) {
      const int i = idx / n, j = idx % n;
      P[idx] = (TB[i * (NP + 1) + j] + TB[(NP + i) * (NP + 1) + j]) + TB[(NP + j) * (NP + 1) + i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

template <int NP>
cudaError_t launch_np(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                      cudaStream_t stream) {
  using C = Cfg<NP>;
  const int64_t tiles = (d + C::KT - 1) / C::KT;
  int grid = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  if (tiles < grid) grid = static_cast<int>(tiles > 0 ? tiles : 1);
  cudaError_t e = cudaFuncSetAttribute(gram_tc_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::SMEM_BYTES);
  if (e != cudaSuccess) return e;
  gram_tc_kernel<NP><<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(rp, n, d, tiles, partials);
  *n_parts = grid;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gram_partials(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                                 int* n_parts, cudaStream_t stream) {
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  if (n <= 32) return launch_np<32>(rp, n, d, partials, num_sms, n_parts, stream);
  return launch_np<64>(rp, n, d, partials, num_sms, n_parts, stream);
}

}  // namespace gar
