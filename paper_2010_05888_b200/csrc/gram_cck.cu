// gram_cck.cu — the pairwise-distance contraction on the CUDA cores for
// kGramCcMaxN < n <= kGramCckMaxN rows: per-CTA partial Gram
// matrices of the centred rows, G_ij = sum_k (x_ik - c_k)(x_jk - c_k), the
// contract of gram_tc.cu / gram_cc.cu.
//
// gram_cc.cu keeps all n(n+1)/2 product sums of a coordinate in one lane,
// which stops at 128 accumulators (n = 15).  Here the upper triangle, in its
// row-major pair order, is cut into K = 2 equal chunks (<= 128 sums each up to
// n = 22): 8 warps = (8/K coordinate parts) x (K chunks); warp w = p*K + c
// computes chunk c over part p of every stage.  (K = 4 for n = 23..31 was
// measured 1.1-2.2x slower than the tensor cores: four different unrolled
// chunk bodies per SM stall on instruction fetch, profiles/r2_gram_cc.md.)  A chunk is a run of whole rows
// i (plus a tail and a head) times all j >= i, so a lane loads only rows from
// the chunk's first row on — about 0.2 shared loads per FFMA — and keeps
// <= 128 fp32 sums.  Two coordinates per lane and step (8-byte loads).
// Every 32 stages (128 coordinates per lane) a butterfly (transpose-)
// reduction over the warp leaves each lane NACC/32 sums, added into fp64;
// parts are summed in fixed order (deterministic).  Precision: <= 128 fp32
// FFMAs + 5 butterfly adds per flushed sum (the tf32 kernel drains 128-product
// TMEM sums), D within 1e-5 of the fp64 oracle.
//
// Ring: all 8 warps synchronise once per stage (named barrier), then refill
// the consumed slot with the stage raw_stages ahead (warp w's lanes issue the
// bulk copies of rows w, w+8, ...).  No producer warp: registers are
// allocated per 4-warp group, and 8 warps leave 255 per thread.
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "gram.h"
#include "gram_common.cuh"

#ifndef GAR_CCK_STEPS
#define GAR_CCK_STEPS 4   // A/B knob (default = product; 2 -> 4: n = 19 0.39 -> 0.31 ms)
#endif

namespace gar {

namespace {

using namespace gram;


template <int N_, bool BF_>
struct CfgK {
  static constexpr int N = N_;
  static constexpr bool BF = BF_;
  static constexpr int K = 2;                           // pair chunks
  static constexpr int WARPS = 8;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int P = WARPS / K;                   // coordinate parts per stage
  static constexpr int NP = (N + 7) / 8 * 8;            // centre pick rows
  static constexpr int ES = BF ? 2 : 4;
  static constexpr int BULK_ALIGN = 16 / ES;
  static constexpr int NPAIR = N * (N + 1) / 2;
  static constexpr int CH = (NPAIR + K - 1) / K;        // pairs per chunk
  // sums per lane: up to 128 padded to a multiple of 32 (all through the
  // butterfly); above, 128 through the butterfly + NREM < 32 reduced one by one
  // (a 160-entry array goes to local memory)
  static constexpr int NBUT = CH <= 128 ? (CH + 31) / 32 * 32 : 128;
  static constexpr int NREM = CH <= 128 ? 0 : CH - 128;
  static constexpr int NACC = NBUT + NREM;
  static constexpr int STEPS = GAR_CCK_STEPS;           // coordinate pairs per lane and stage
  static constexpr int PART = 64 * STEPS;               // coordinates per warp and stage
  static constexpr int RAW_KT = P * PART;
  static constexpr int FLUSH_ST = 128 / (2 * STEPS);    // 128 coordinates per lane between flushes
  static constexpr int RAW_PITCH = RAW_KT * ES + 16;
  static constexpr int RAW_STAGES_MAX = 8;
  static constexpr int PICK = center_pick_bytes(NP);
  static constexpr int WSUM = WARPS * NACC * 8;
  static constexpr int SCRATCH = PICK > WSUM ? PICK : WSUM;   // wsum aliases the pick scratch
  static constexpr int SMEM_BYTES = 227 * 1024;
  static constexpr int BAR_BYTES = RAW_STAGES_MAX * 8 + 16;
  static constexpr int RAW_REGION = SMEM_BYTES - 128 - SCRATCH - BAR_BYTES;
  static_assert(NREM < 32, "at most 159 sums per lane");
  static_assert(RAW_REGION >= 2 * N * RAW_PITCH, "two raw stages");
};

// index of pair (i, j), i <= j, in row-major upper-triangle order
__host__ __device__ constexpr int pair_index(int n, int i, int j) { return i * n - i * (i - 1) / 2 + (j - i); }

// first row with a pair in [e, ...): the row of pair index e
constexpr int row_of_pair(int n, int e) {
  int i = 0;
  while (i + 1 < n && pair_index(n, i + 1, i + 1) <= e) ++i;
  return i;
}

template <bool BF>
__device__ __forceinline__ float2 ld_pair2(const unsigned char* row, int k) {
  if constexpr (BF) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 2 * k);
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  } else {
    return *reinterpret_cast<const float2*>(row + 4 * k);
  }
}

template <bool BF>
__device__ __forceinline__ float ld_one1(const unsigned char* row, int k) {
  if constexpr (BF) {
    return bf16_to_f32(*reinterpret_cast<const unsigned short*>(row + 2 * k));
  } else {
    return *reinterpret_cast<const float*>(row + 4 * k);
  }
}

// acc += the chunk's products of one coordinate's centred values h[R0..N)
template <int N, int LO, int HI, int R0>
__device__ __forceinline__ void chunk_fma(float* acc, const float* h) {
#pragma unroll
  for (int i = R0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      const int e = pair_index(N, i, j);
      if (e >= LO && e < HI) acc[e - LO] = fmaf(h[i - R0], h[j - R0], acc[e - LO]);
    }
}

template <int NACC>
__device__ __forceinline__ void flush_k(float* acc, double* acc64, int lane) {
#pragma unroll
  for (int o = 16, half = NACC / 2; o >= 1; o >>= 1, half >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int e = 0; e < half; ++e) {
      const float send = up ? acc[e] : acc[e + half];
      const float keep = up ? acc[e + half] : acc[e];
      acc[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
#pragma unroll
  for (int t = 0; t < NACC / 32; ++t) acc64[t] += static_cast<double>(acc[t]);
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.f;
}

struct SliceK {
  int64_t k_begin, k_end, S, d_bulk;
};

template <int N, bool BF>
__device__ __forceinline__ void issue_stage_k(const RowPtrs& rows, const SliceK& sl, unsigned char* slot, uint64_t* bar,
                                              int64_t j, int warp, int lane, uint64_t pol, int l2_hint) {
  using C = CfgK<N, BF>;
  const int64_t k0 = sl.k_begin + j * C::RAW_KT;
  const int64_t cnt = (sl.k_end - k0 < C::RAW_KT) ? sl.k_end - k0 : C::RAW_KT;
  const uint32_t bytes = static_cast<uint32_t>(cnt & ~int64_t(C::BULK_ALIGN - 1)) * C::ES;
  const int my_rows = (N > warp) ? (N - warp + C::WARPS - 1) / C::WARPS : 0;
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes * static_cast<uint32_t>(my_rows));
  __syncwarp();
  const int r = warp + C::WARPS * lane;
  if (bytes && r < N) {
    const void* src = reinterpret_cast<const unsigned char*>(rows.p[r]) + k0 * C::ES;
    if (l2_hint) bulk_g2s(slot + r * C::RAW_PITCH, src, bytes, bar, pol);
    else bulk_g2s_plain(slot + r * C::RAW_PITCH, src, bytes, bar);
  }
}

// one warp: chunk CK over coordinate part `part` of every stage of the slice
template <int N, bool BF, int CK>
__device__ __forceinline__ void consume_k(const RowPtrs& rows, const SliceK& sl, unsigned char* raw, int raw_bytes,
                                          int raw_stages, uint64_t* full, int rc, double* wsum, int warp, int lane,
                                          int part, int l2_hint) {
  using C = CfgK<N, BF>;
  constexpr int LO = CK * C::CH;
  constexpr int HI = (CK + 1) * C::CH < C::NPAIR ? (CK + 1) * C::CH : C::NPAIR;
  constexpr int R0 = row_of_pair(N, LO);               // first row the chunk multiplies
  constexpr int NL = N - R0;                           // rows loaded
  const uint64_t pol = policy_evict_first();
  float acc[C::NACC];
#pragma unroll
  for (int e = 0; e < C::NACC; ++e) acc[e] = 0.f;
  double acc64[C::NBUT / 32];
#pragma unroll
  for (int t = 0; t < C::NBUT / 32; ++t) acc64[t] = 0.0;
  double accr = 0.0;                                   // remainder entry NBUT + lane (lane < NREM)
  for (int64_t j = 0; j < sl.S && j < raw_stages; ++j)
    issue_stage_k<N, BF>(rows, sl, raw + j * raw_bytes, &full[j], j, warp, lane, pol, l2_hint);
  int rs = 0, fl = 0;
  uint32_t ph = 0;
  for (int64_t j = 0; j < sl.S; ++j) {
    const int64_t k0 = sl.k_begin + j * C::RAW_KT;
    unsigned char* st = raw + rs * raw_bytes;
    mbar_wait(&full[rs], ph);
    const unsigned char* rR = st + R0 * C::RAW_PITCH;
    const unsigned char* rC = st + rc * C::RAW_PITCH;
    const int kb = part * C::PART;
    if (k0 + C::RAW_KT <= sl.d_bulk) {               // a full stage, all of it in the ring
#pragma unroll 1
      for (int t = 0; t < C::STEPS; ++t) {            // rolled: the K chunk bodies share the I-cache
        const int k = kb + 2 * lane + 64 * t;
        const float2 c2 = ld_pair2<BF>(rC, k);
        const float cx = fin(c2.x), cy = fin(c2.y);
        float2 v[NL];
#pragma unroll
        for (int a = 0; a < NL; ++a) v[a] = ld_pair2<BF>(rR + a * C::RAW_PITCH, k);
        float h[NL];
#pragma unroll
        for (int a = 0; a < NL; ++a) h[a] = __fsub_rn(v[a].x, cx);
        chunk_fma<N, LO, HI, R0>(acc, h);
#pragma unroll
        for (int a = 0; a < NL; ++a) h[a] = __fsub_rn(v[a].y, cy);
        chunk_fma<N, LO, HI, R0>(acc, h);
      }
    } else {                                         // the slice's last stage: ragged, tail from global
      const int cnt = static_cast<int>((sl.k_end - k0 < C::RAW_KT) ? sl.k_end - k0 : C::RAW_KT);
      const int ke = (kb + C::PART < cnt) ? kb + C::PART : cnt;
      using E = Elem<typename std::conditional<BF, bf2, float>::type>;
      for (int k = kb + lane; k < ke; k += 32) {
        const bool ring = k0 + k < sl.d_bulk;
        auto val = [&](int r) {
          return ring ? ld_one1<BF>(st + r * C::RAW_PITCH, k) : E::value(rows.p[r], k0 + k);
        };
        const float c = fin(val(rc));
        float h[NL];
#pragma unroll
        for (int a = 0; a < NL; ++a) h[a] = __fsub_rn(val(R0 + a), c);
        chunk_fma<N, LO, HI, R0>(acc, h);
      }
    }
    named_bar(4, C::THREADS);                         // stage j consumed by every warp
    if (j + raw_stages < sl.S)
      issue_stage_k<N, BF>(rows, sl, st, &full[rs], j + raw_stages, warp, lane, pol, l2_hint);
    if (++fl == C::FLUSH_ST || j + 1 == sl.S) {
      flush_k<C::NBUT>(acc, acc64, lane);
#pragma unroll
      for (int e = 0; e < C::NREM; ++e) {              // fixed xor tree: every lane holds the sum
        float v = acc[C::NBUT + e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == e) accr += static_cast<double>(v);
        acc[C::NBUT + e] = 0.f;
      }
      fl = 0;
    }
    if (++rs == raw_stages) rs = 0, ph ^= 1;
  }
  int eb = 0;
  for (int o = 16, half = C::NBUT / 2; o >= 1; o >>= 1, half >>= 1) eb += (lane & o) ? half : 0;
  // wsum aliases the centre-pick scratch, free since the kernel's __syncthreads
#pragma unroll
  for (int t = 0; t < C::NBUT / 32; ++t) wsum[warp * C::NACC + eb + t] = acc64[t];
  if (lane < C::NREM) wsum[warp * C::NACC + C::NBUT + lane] = accr;
}

template <int N, bool BF, int CK = 0>
__device__ __forceinline__ void consume_dispatch(int ck, const RowPtrs& rows, const SliceK& sl, unsigned char* raw,
                                                 int raw_bytes, int raw_stages, uint64_t* full, int rc, double* wsum,
                                                 int warp, int lane, int part, int l2_hint) {
  if constexpr (CK < CfgK<N, BF>::K) {
    if (ck == CK)
      consume_k<N, BF, CK>(rows, sl, raw, raw_bytes, raw_stages, full, rc, wsum, warp, lane, part, l2_hint);
    else
      consume_dispatch<N, BF, CK + 1>(ck, rows, sl, raw, raw_bytes, raw_stages, full, rc, wsum, warp, lane, part,
                                      l2_hint);
  }
}

template <int N, bool BF>
__global__ void __launch_bounds__(CfgK<N, BF>::THREADS, 1)
    gram_cck_kernel(const __grid_constant__ RowPtrs rows, int64_t d, double* __restrict__ partials, int l2_hint,
                    int raw_stages, int raw_bytes) {
  using C = CfgK<N, BF>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  unsigned char* raw = base;
  unsigned char* scratch = raw + C::RAW_REGION;
  double* wsum = reinterpret_cast<double*>(scratch);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + C::SCRATCH);   // [RAW_STAGES_MAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  SliceK sl;
  const int64_t nst = (d + C::RAW_KT - 1) / C::RAW_KT;
  const int64_t s0 = nst * blockIdx.x / gridDim.x;
  sl.S = nst * (blockIdx.x + 1) / gridDim.x - s0;
  sl.k_begin = s0 * C::RAW_KT;
  sl.k_end = ((s0 + sl.S) * C::RAW_KT < d) ? (s0 + sl.S) * C::RAW_KT : d;
  sl.d_bulk = d & ~int64_t(C::BULK_ALIGN - 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < raw_stages; ++s) mbar_init(&full[s], C::WARPS);
    fence_mbar_init();
  }
  const int rc = center_pick<C::THREADS, C::NP, BF>(rows, N, d, sl.k_begin, scratch);
  __syncthreads();                                   // barriers initialised; the pick scratch is free again

  consume_dispatch<N, BF>(warp % C::K, rows, sl, raw, raw_bytes, raw_stages, full, rc, wsum, warp, lane,
                          warp / C::K, l2_hint);
  named_bar(3, C::THREADS);
  double* Pm = partials + static_cast<size_t>(blockIdx.x) * N * N;
  for (int idx = threadIdx.x; idx < N * N; idx += C::THREADS) {
    int i = idx / N, jj = idx % N;
    if (i > jj) {
      const int t = i; i = jj; jj = t;
    }
    const int e = pair_index(N, i, jj), ck = e / C::CH, off = e - ck * C::CH;
    double s = 0.0;
    for (int p = 0; p < C::P; ++p) s += wsum[(p * C::K + ck) * C::NACC + off];
    Pm[idx] = s;
  }
}

template <int N, bool BF>
cudaError_t launch_cck(const RowPtrs& rp, int64_t d, double* partials, int num_sms, int* n_parts,
                       cudaStream_t stream) {
  using C = CfgK<N, BF>;
  const int64_t nst = (d + C::RAW_KT - 1) / C::RAW_KT;
  int grid = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  if (nst < grid) grid = static_cast<int>(nst > 0 ? nst : 1);
  int occ = 0;
  auto kern = gram_cck_kernel<N, BF>;
  cudaError_t e = cached_occupancy(kern, C::THREADS, C::SMEM_BYTES, &occ);
  if (e != cudaSuccess) return e;
  const int raw_bytes = N * C::RAW_PITCH;
  int raw_stages = C::RAW_REGION / raw_bytes;
  if (raw_stages > C::RAW_STAGES_MAX) raw_stages = C::RAW_STAGES_MAX;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(rp, d, partials, l2_evict_first_enabled(), raw_stages,
                                                     raw_bytes);
  *n_parts = grid;
  return cudaGetLastError();
}

template <int LO, int HI, bool BF>
cudaError_t dispatch_cck(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                         cudaStream_t stream) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (n == LO) return launch_cck<LO, BF>(rp, d, partials, num_sms, n_parts, stream);
    return dispatch_cck<LO + 1, HI, BF>(rp, n, d, partials, num_sms, n_parts, stream);
  }
}

}  // namespace

cudaError_t launch_gram_cck(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                            int* n_parts, cudaStream_t stream, int dtype) {
  if (n <= kGramCcMaxN || n > kGramCckLimit) return cudaErrorInvalidValue;
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
  return dtype == kBF16
             ? dispatch_cck<kGramCcMaxN + 1, kGramCckLimit, true>(rp, n, d, partials, num_sms, n_parts, stream)
             : dispatch_cck<kGramCcMaxN + 1, kGramCckLimit, false>(rp, n, d, partials, num_sms, n_parts, stream);
}

}  // namespace gar
