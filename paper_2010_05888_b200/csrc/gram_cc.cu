// gram_cc.cu — the pairwise-distance contraction on the CUDA cores (FFMA) for
// small n (row a5 of DESIGN.md §1; §4.2c): per-CTA partial Gram matrices of the
// centred rows, G_ij = sum_k (x_ik - c_k)(x_jk - c_k), same contract as
// gram_tc.cu.
//
// Why: for small n the tensor-core kernel is bound by per-tile costs that do
// not shrink with n (the 128 x 64 MMA operands over padded rows, the tf32
// hi/lo stores: 28+ bytes of shared-memory traffic per element) while the
// arithmetic is tiny: n(n+1)/2 products per coordinate (66 at n = 11).  Here
// every element crosses shared memory twice (TMA write, one read) and is
// multiplied in fp32 FFMA (one rounding per product-add, more accurate than
// the tf32 split).
//
// Layout (n <= 15, every loop unrolled for the exact n): each element is read
// from the TMA ring once; a lane keeps all n(n+1)/2 products-sums of the
// coordinates it visits (consumer warp w owns part w of every raw stage, lane
// l its coordinates l, l+32, ...), in fp32 over FLUSH_ST stages (128 coordinates
// per lane); then a butterfly (transpose-)reduction over the 32 lanes leaves
// each lane NACC/32 of the entries, added into fp64; warps are summed in fixed
// order at the end (deterministic).  Precision: <= 128 fp32 FFMAs per lane plus
// 5 butterfly levels before each fp64 add, i.e. <= ~133 * 2^-24 of the flushed
// |products|, the class of the tf32 kernel's 128-product TMEM drains (measured
// D errors ~1e-8 relative, tools/check_gram.py).
#include <cmath>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "gram.h"
#include "gram_common.cuh"

#ifndef GAR_CC_FLUSH
#define GAR_CC_FLUSH 32   // A/B knob (default = product; 8 -> 32: n = 15 0.256 -> 0.246 ms)
#endif

namespace gar {

namespace {

using namespace gram;

template <int N_, bool BF_>
struct CfgCC {
  static constexpr int N = N_;                    // rows (exact: every loop below is unrolled)
  static constexpr int NP = (N + 7) / 8 * 8;      // padded rows (centre pick, ring rows)
  static constexpr bool BF = BF_;
  static constexpr int ES = BF ? 2 : 4;
  static constexpr int BULK_ALIGN = 16 / ES;
  static constexpr int NPAIR = N * (N + 1) / 2;   // upper triangle incl. the diagonal
  static constexpr int NACC = (NPAIR + 31) / 32 * 32;   // accumulators per lane (butterfly needs 32 | NACC)
  // registers are allocated per 4-warp group: 15 warps leave 128 per thread
  // (<= 96 accumulators, n <= 12); 8 warps leave 255 (<= 128, n <= 15)
  static constexpr int CONS_WARPS = N <= 12 ? 12 : 7;   // coordinate parts of a stage, one per warp
  static constexpr int PROD_WARPS = N <= 12 ? 3 : 1;
  static constexpr int THREADS = (CONS_WARPS + PROD_WARPS) * 32;
  static constexpr int RAW_KT = CONS_WARPS * 128;       // coordinates per raw stage
  static constexpr int PART = RAW_KT / CONS_WARPS;      // 128 coordinates per warp and stage
  static constexpr int PER_LANE = PART / 32;            // 4
  static constexpr int FLUSH_ST = GAR_CC_FLUSH;   // stages summed in fp32 per lane (4 coordinates each)
  static constexpr int RAW_PITCH = RAW_KT * ES + 16;
  static constexpr int RAW_STAGES_MAX = 8;
  static constexpr int SCRATCH = center_pick_bytes(NP);   // centre pick
  static constexpr int WSUM_BYTES = CONS_WARPS * NACC * 8;                    // per-warp fp64 sums
  static constexpr int SMEM_BYTES = 227 * 1024;
  static constexpr int BAR_BYTES = (PROD_WARPS + 1) * RAW_STAGES_MAX * 8 + 16;
  static constexpr int RAW_REGION = SMEM_BYTES - 128 - SCRATCH - WSUM_BYTES - BAR_BYTES;
  static_assert(N >= 1 && NACC <= 128, "one accumulator set of <= 128 per lane");
  static_assert(RAW_KT % (32 * CONS_WARPS) == 0, "work split");
  static_assert(RAW_REGION >= 2 * NP * RAW_PITCH, "two raw stages");
};

// one coordinate value of a ring row at offset k (fp32 or widened bf16)
template <bool BF>
__device__ __forceinline__ float ld_raw(const unsigned char* row, int k) {
  if constexpr (BF) {
    return bf16_to_f32(*reinterpret_cast<const unsigned short*>(row + 2 * k));
  } else {
    return *reinterpret_cast<const float*>(row + 4 * k);
  }
}

template <int N, bool BF>
__global__ void __launch_bounds__(CfgCC<N, BF>::THREADS, 1)
    gram_cc_kernel(const __grid_constant__ RowPtrs rows, int64_t d, double* __restrict__ partials, int l2_hint,
                   int raw_stages, int raw_bytes) {
  using C = CfgCC<N, BF>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  unsigned char* raw = base;                                              // raw_stages x [NP][RAW_PITCH]
  unsigned char* scratch = raw + C::RAW_REGION;                           // centre pick
  double* wsum = reinterpret_cast<double*>(scratch + C::SCRATCH);         // [CONS_WARPS][NACC]
  uint64_t* full = reinterpret_cast<uint64_t*>(wsum + C::CONS_WARPS * C::NACC);   // [RAW_STAGES_MAX][PROD_WARPS]
  uint64_t* empty = full + C::RAW_STAGES_MAX * C::PROD_WARPS;            // [RAW_STAGES_MAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // contiguous, balanced coordinate range of this CTA, in whole raw stages
  const int64_t nst = (d + C::RAW_KT - 1) / C::RAW_KT;
  const int64_t s0 = nst * blockIdx.x / gridDim.x;
  const int64_t S = nst * (blockIdx.x + 1) / gridDim.x - s0;
  const int64_t k_begin = s0 * C::RAW_KT;
  const int64_t k_end = ((s0 + S) * C::RAW_KT < d) ? (s0 + S) * C::RAW_KT : d;

  if (threadIdx.x == 0) {
    for (int s = 0; s < raw_stages; ++s) {
      for (int q = 0; q < C::PROD_WARPS; ++q) mbar_init(&full[s * C::PROD_WARPS + q], 1);
      mbar_init(&empty[s], C::CONS_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= C::CONS_WARPS) {
    // ====================================================== TMA producers
    const int q = warp - C::CONS_WARPS;
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int my_rows = (N > q) ? (N - q + C::PROD_WARPS - 1) / C::PROD_WARPS : 0;
      int rs = 0;
      uint32_t use = 0;
      for (int64_t j = 0; j < S; ++j, (++rs == raw_stages) ? (rs = 0, ++use) : 0) {
        if (use > 0) mbar_wait_sleep(&empty[rs], (use - 1) & 1);
        const int64_t k0 = k_begin + j * C::RAW_KT;
        const int64_t cnt = (k_end - k0 < C::RAW_KT) ? k_end - k0 : C::RAW_KT;
        const uint32_t bytes = static_cast<uint32_t>(cnt & ~int64_t(C::BULK_ALIGN - 1)) * C::ES;
        uint64_t* bar = &full[rs * C::PROD_WARPS + q];
        mbar_arrive_expect_tx(bar, bytes * static_cast<uint32_t>(my_rows));
        if (bytes) {
          unsigned char* dst = raw + rs * raw_bytes;
          for (int r = q; r < N; r += C::PROD_WARPS) {
            const void* src = reinterpret_cast<const unsigned char*>(rows.p[r]) + k0 * C::ES;
            if (l2_hint) bulk_g2s(dst + r * C::RAW_PITCH, src, bytes, bar, pol);
            else bulk_g2s_plain(dst + r * C::RAW_PITCH, src, bytes, bar);
          }
        }
      }
    }
    return;
  }

  // ======================================================== consumers
  constexpr int NT = C::CONS_WARPS * 32;
  const int rc = center_pick<NT, C::NP, BF>(rows, N, d, k_begin, scratch);
  double acc64[C::NACC / 32];                               // this lane's entries after the butterfly
#pragma unroll
  for (int t = 0; t < C::NACC / 32; ++t) acc64[t] = 0.0;
  const int64_t d_bulk = d & ~int64_t(C::BULK_ALIGN - 1);
  float acc[C::NACC];
#pragma unroll
  for (int e = 0; e < C::NACC; ++e) acc[e] = 0.f;
  using E = Elem<typename std::conditional<BF, bf2, float>::type>;
  int rs = 0;
  uint32_t rphase = 0;
  for (int64_t j = 0; j < S; ++j, (++rs == raw_stages) ? (rs = 0, rphase ^= 1) : 0) {
#pragma unroll
    for (int q = 0; q < C::PROD_WARPS; ++q) mbar_wait(&full[rs * C::PROD_WARPS + q], rphase);
    const int64_t k0 = k_begin + j * C::RAW_KT;
    const int cnt = static_cast<int>((k_end - k0 < C::RAW_KT) ? k_end - k0 : C::RAW_KT);
    const unsigned char* st = raw + rs * raw_bytes;
    const int kb = warp * C::PART;
    const int ke = (kb + C::PART < cnt) ? kb + C::PART : cnt;
    // one coordinate: centre, the N centred values, the N(N+1)/2 products.
    // DIRECT: read from global memory (the < BULK_ALIGN coordinates past the
    // last bulk copy of the vector)
    auto coord = [&](int k, auto direct_tag) {
      constexpr bool DIRECT = decltype(direct_tag)::value;
      auto load = [&](int r) {
        if constexpr (DIRECT) return E::value(rows.p[r], k0 + k);
        else return ld_raw<BF>(st + r * C::RAW_PITCH, k);
      };
      const float c = fin(load(rc));
      float h[N];
#pragma unroll
      for (int a = 0; a < N; ++a) h[a] = __fsub_rn(load(a), c);
      int e = 0;
#pragma unroll
      for (int a = 0; a < N; ++a)
#pragma unroll
        for (int bb = a; bb < N; ++bb, ++e) acc[e] = fmaf(h[a], h[bb], acc[e]);
    };
    if (k0 + ke <= d_bulk) {                                  // the whole part came by bulk copy
#pragma unroll
      for (int t = 0; t < C::PER_LANE; ++t) {
        const int k = kb + lane + 32 * t;
        if (k < ke) coord(k, std::false_type{});
      }
    } else {
      for (int k = kb + lane; k < ke; k += 32) {
        if (k0 + k < d_bulk) coord(k, std::false_type{});
        else coord(k, std::true_type{});
      }
    }
    // release the stage before any reduction (the sums are in registers)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[rs]);
    if ((j + 1) % C::FLUSH_ST != 0 && j + 1 != S) continue;
    // butterfly transpose-reduction over the 32 lanes: after the step with
    // offset o each lane keeps the half of its values selected by (lane & o),
    // summed with the partner's; NACC -> NACC / 32 values per lane
#pragma unroll
    for (int o = 16, half = C::NACC / 2; o >= 1; o >>= 1, half >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int e = 0; e < half; ++e) {
        const float send = up ? acc[e] : acc[e + half];
        const float keep = up ? acc[e + half] : acc[e];
        acc[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
#pragma unroll
    for (int t = 0; t < C::NACC / 32; ++t) acc64[t] += static_cast<double>(acc[t]);
#pragma unroll
    for (int e = 0; e < C::NACC; ++e) acc[e] = 0.f;
  }
  // the entries acc64[t] stand for: e = t + sum over o of ((lane & o) ? half(o) : 0)
  int ebase = 0;
#pragma unroll
  for (int o = 16, half = C::NACC / 2; o >= 1; o >>= 1, half >>= 1) ebase += (lane & o) ? half : 0;
#pragma unroll
  for (int t = 0; t < C::NACC / 32; ++t) wsum[warp * C::NACC + ebase + t] = acc64[t];
  named_bar(3, NT);
  // per-CTA partial: pair (i <= j) -> entry e of the upper triangle, warps
  // summed in fixed order
  double* Pm = partials + static_cast<size_t>(blockIdx.x) * N * N;
  for (int idx = threadIdx.x; idx < N * N; idx += NT) {
    int i = idx / N, jj = idx % N;
    if (i > jj) {
      const int t = i; i = jj; jj = t;
    }
    const int e = i * N - i * (i - 1) / 2 + (jj - i);
    double s = 0.0;
    for (int w = 0; w < C::CONS_WARPS; ++w) s += wsum[w * C::NACC + e];
    Pm[idx] = s;
  }
}

template <int N, bool BF>
cudaError_t launch_cc(const RowPtrs& rp, int64_t d, double* partials, int num_sms, int* n_parts,
                      cudaStream_t stream) {
  using C = CfgCC<N, BF>;
  const int64_t nst = (d + C::RAW_KT - 1) / C::RAW_KT;
  int grid = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  if (nst < grid) grid = static_cast<int>(nst > 0 ? nst : 1);
  int occ = 0;
  auto kern = gram_cc_kernel<N, BF>;
  cudaError_t e = cached_occupancy(kern, C::THREADS, C::SMEM_BYTES, &occ);
  if (e != cudaSuccess) return e;
  const int raw_bytes = C::NP * C::RAW_PITCH;
  int raw_stages = C::RAW_REGION / raw_bytes;
  if (raw_stages > C::RAW_STAGES_MAX) raw_stages = C::RAW_STAGES_MAX;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(rp, d, partials, l2_evict_first_enabled(), raw_stages,
                                                     raw_bytes);
  *n_parts = grid;
  return cudaGetLastError();
}

template <int LO, int HI, bool BF>
cudaError_t dispatch_cc(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                        cudaStream_t stream) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (n == LO) return launch_cc<LO, BF>(rp, d, partials, num_sms, n_parts, stream);
    return dispatch_cc<LO + 1, HI, BF>(rp, n, d, partials, num_sms, n_parts, stream);
  }
}

}  // namespace

cudaError_t launch_gram_cc(const float* const* rows, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                           cudaStream_t stream, int dtype) {
  if (n < 1 || n > kGramCcMaxN) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  return dtype == kBF16 ? dispatch_cc<1, kGramCcMaxN, true>(rp, n, d, partials, num_sms, n_parts, stream)
                        : dispatch_cc<1, kGramCcMaxN, false>(rp, n, d, partials, num_sms, n_parts, stream);
}

}  // namespace gar
