// gram_ccb.cuh — the pairwise-distance contraction on the CUDA cores for
// kGramCcbMinN <= n <= kGramCcbMaxN rows (33..36): per-CTA
// partial Gram matrices of the centred rows, G_ij = sum_k (x_ik - c_k)(x_jk -
// c_k), the contract of gram_tc.cu / gram_cc.cu.
//
// Why: from 33 rows the tensor-core Gram pads to NP = 64 and is bound by the
// N = 64 MMA issue cost and its padded operand traffic (1.27 ms at n = 35
// against 0.55 ms of HBM time).  Here the n(n+1)/2 products per coordinate run
// as FFMA: 1.05 ms at S = 9 (n = 33..36); from S = 10 (n >= 37) and below
// n = 33 the tensor cores win again (profiles/r2_gram_cc.md).
//
// Register blocking.  Rows in 4 groups of S = ceil(n/4) (the last group padded
// with zero rows that live in every ring slot); the upper triangle of G in 8
// units: warps 0..5 the off-diagonal S x S group blocks, warps 6 and 7 two
// diagonal triangles each ({1, 2}, {0, 3}).  A warp owns its unit over EVERY
// coordinate of the CTA's slice; a lane keeps the unit's products in fp32
// registers, loads the unit's rows for two coordinates at a time (8-byte
// shared loads, conflict-free) and issues S*S FFMA per coordinate.  Only two
// code paths (block, triangle pair) with the group offsets as runtime values:
// 8 different unrolled bodies thrash the instruction cache (measured: 10x
// slower, "no instruction" stalls).  Every FLUSH_ST stages (128 coordinates
// per lane) a butterfly (transpose-)reduction over the 32 lanes leaves each
// lane NACC/32 sums, added into fp64 registers.  Precision: <= 128 fp32 FFMAs +
// 5 butterfly adds per flushed sum, the error class of the tf32 kernel's
// 128-product TMEM drains (D within 1e-5 of the fp64 oracle; measured ~1e-8,
// tools/check_gram.py).  Deterministic: fixed warp/lane/stage order, fixed CTA
// order in gram_reduce_kernel.
#pragma once
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "gram.h"
#include "gram_common.cuh"

#ifndef GAR_CCB_KT
#define GAR_CCB_KT 512
#endif

namespace gar {
namespace ccb {

using namespace gram;

template <int N, bool BF_>
struct Cfg {
  static constexpr bool BF = BF_;
  static constexpr int S = (N + 3) / 4;                      // rows per group
  static constexpr int NR = 4 * S;                           // ring rows per slot (N real + zero rows)
  static constexpr int NP = (N + 7) / 8 * 8;                 // centre pick rows
  static constexpr int ES = BF ? 2 : 4;
  static constexpr int BULK_ALIGN = 16 / ES;
  static constexpr int WARPS = 8;                            // every warp computes a unit and issues copies
  static constexpr int THREADS = WARPS * 32;
  static constexpr int NACC_OFF = (S * S + 31) / 32 * 32;        // block unit accumulators
  static constexpr int NACC_DIAG = (S * (S + 1) + 31) / 32 * 32;  // triangle-pair unit accumulators
  static constexpr int RAW_KT = GAR_CCB_KT;                  // coordinates per stage
  static constexpr int PER_LANE = RAW_KT / 64;               // coordinate pairs per lane and stage
  static constexpr int FLUSH_ST = 128 * 32 / RAW_KT;         // 128 coordinates per lane between flushes
  static constexpr int RAW_PITCH = RAW_KT * ES + 16;
  static constexpr int RAW_STAGES_MAX = 8;
  static constexpr int PICK = center_pick_bytes(NP);                      // centre pick scratch
  static constexpr int WSUM = WARPS * NACC_DIAG * 8;                      // fp64 unit sums (aliases PICK)
  static constexpr int SCRATCH = PICK > WSUM ? PICK : WSUM;
  static constexpr int SMEM_BYTES = 227 * 1024;
  static constexpr int BAR_BYTES = RAW_STAGES_MAX * 8 + 16;
  static constexpr int RAW_REGION = SMEM_BYTES - 128 - SCRATCH - BAR_BYTES;
  static_assert(N - 3 * S >= 1, "4 non-empty groups");
  static_assert(RAW_REGION >= 2 * NR * RAW_PITCH, "two raw stages");
};

// unit of warp w: 0..5 the blocks (0,1) (0,2) (0,3) (1,2) (1,3) (2,3); 6 the
// triangles of groups 1 and 2, 7 those of groups 0 and 3 (warps w and w+4 share
// an SM sub-partition: 6 and 7 pair with the blocks of warps 2 and 3)
__device__ __forceinline__ int unit_gi(int w) { return w < 3 ? 0 : w < 5 ? 1 : w == 5 ? 2 : w == 6 ? 1 : 0; }
__device__ __forceinline__ int unit_gj(int w) { return w == 0 ? 1 : (w == 1 || w == 3 || w == 6) ? 2 : 3; }

// two consecutive coordinates (k even) of a ring row, widened to fp32
template <bool BF>
__device__ __forceinline__ float2 ld_pair(const unsigned char* row, int k) {
  if constexpr (BF) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(row + 2 * k);
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
  } else {
    return *reinterpret_cast<const float2*>(row + 4 * k);
  }
}

template <bool BF>
__device__ __forceinline__ float ld_one(const unsigned char* row, int k) {
  if constexpr (BF) {
    return bf16_to_f32(*reinterpret_cast<const unsigned short*>(row + 2 * k));
  } else {
    return *reinterpret_cast<const float*>(row + 4 * k);
  }
}

// acc += the unit's products of one coordinate's centred rows hI, hJ (S each):
// the block hI x hJ, or the upper triangles of hI and of hJ
template <int S, bool DIAG>
__device__ __forceinline__ void unit_fma(float* acc, const float* hI, const float* hJ) {
  if constexpr (DIAG) {
    int e = 0;
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = a; b < S; ++b, ++e) acc[e] = fmaf(hI[a], hI[b], acc[e]);
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = a; b < S; ++b, ++e) acc[e] = fmaf(hJ[a], hJ[b], acc[e]);
  } else {
#pragma unroll
    for (int a = 0; a < S; ++a)
#pragma unroll
      for (int b = 0; b < S; ++b) acc[a * S + b] = fmaf(hI[a], hJ[b], acc[a * S + b]);
  }
}

// butterfly (transpose-)reduction of NACC lane values over the warp, then
// into fp64: after the step with offset o a lane keeps the half of its values
// selected by (lane & o), summed with its partner's
template <int NACC>
__device__ __forceinline__ void flush(float* acc, double* acc64, int lane) {
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

// entry of acc64[t] on lane `lane` after the butterfly: flush_base + t
__device__ __forceinline__ int flush_base(int nacc, int lane) {
  int e = 0;
  for (int o = 16, half = nacc / 2; o >= 1; o >>= 1, half >>= 1) e += (lane & o) ? half : 0;
  return e;
}

struct Slice {
  int64_t k_begin, k_end, S, d_bulk;
};

// Pre-centring (fp32 rows, GAR_CCB_PRE): the warps first rewrite the landed
// stage in place, x <- x - c (warp w its 1/8 of the coordinates, 16-byte
// shared accesses), so the unit loops load centred values: per coordinate
// 1.5 n instructions instead of one FSUB per unit row (4 n).  Same arithmetic
// (one __fsub_rn per element), bit-identical result.
#ifndef GAR_CCB_PRE
#define GAR_CCB_PRE 0
#endif

template <int N>
__device__ __forceinline__ void centre_slice(unsigned char* st, int rc, int cnt_ring, int warp, int lane) {
  using C = Cfg<N, false>;
  constexpr int SL = C::RAW_KT / C::WARPS;        // coordinates of this warp
  constexpr int CH = SL / 4;                      // 16-byte chunks per row
  constexpr int RG = 32 / CH;                     // row groups over the lanes
  static_assert(SL % 4 == 0 && 32 % CH == 0, "slice geometry");
  const int p = lane % CH, q = lane / CH;
  const int k = warp * SL + 4 * p;
  const bool live = k < cnt_ring;                 // cnt_ring is a multiple of 4
  float4 c = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live) {
    c = *reinterpret_cast<const float4*>(st + rc * C::RAW_PITCH + 4 * k);
    c = make_float4(fin(c.x), fin(c.y), fin(c.z), fin(c.w));
  }
  __syncwarp();                                   // every lane holds c before row rc is rewritten
  if (live) {
#pragma unroll
    for (int r = q; r < N; r += RG) {
      float4* x = reinterpret_cast<float4*>(st + r * C::RAW_PITCH + 4 * k);
      float4 v = *x;
      v.x = __fsub_rn(v.x, c.x);
      v.y = __fsub_rn(v.y, c.y);
      v.z = __fsub_rn(v.z, c.z);
      v.w = __fsub_rn(v.w, c.w);
      *x = v;
    }
  }
  fence_proxy_async_smem();                       // these generic writes precede the slot's next bulk copy
}

// Ring: raw_stages slots of one stage each.  All 8 warps synchronise once per
// stage (named barrier): after it stage j is consumed by everyone (and, with
// pre-centring, stage j+1 centred), so its slot is refilled at once with stage
// j + raw_stages: warp w's lanes issue the bulk copies of rows w, w+8, ...,
// lane 0 first posting their bytes on the slot's full barrier (8 arrivals per
// phase).  No producer warp: register allocation is per 4-warp group, and 8
// warps leave each thread up to 255 registers for the unit's accumulators.
template <int N, bool BF>
__device__ __forceinline__ void issue_stage(const RowPtrs& rows, const Slice& sl, unsigned char* slot, uint64_t* bar,
                                            int64_t j, int warp, int lane, uint64_t pol, int l2_hint) {
  using C = Cfg<N, BF>;
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

// one warp: its unit (rows I0.., J0.., S each) over every coordinate of the slice
template <int N, bool BF, bool DIAG>
__device__ __forceinline__ void consume(const RowPtrs& rows, const Slice& sl, unsigned char* raw, int raw_bytes,
                                        int raw_stages, uint64_t* full, int rc, double* wsum, int warp, int lane,
                                        int l2_hint, int I0, int J0) {
  using C = Cfg<N, BF>;
  constexpr int S = C::S;
  constexpr int NACC = DIAG ? C::NACC_DIAG : C::NACC_OFF;
  constexpr bool PRE = !BF && GAR_CCB_PRE;
  constexpr int NT = C::THREADS;
  const uint64_t pol = policy_evict_first();
  float acc[NACC];
#pragma unroll
  for (int e = 0; e < NACC; ++e) acc[e] = 0.f;
  double acc64[NACC / 32];
#pragma unroll
  for (int t = 0; t < NACC / 32; ++t) acc64[t] = 0.0;
  auto ring_count = [&](int64_t k0) {             // coordinates of stage k0.. that came by bulk copy
    const int64_t e = sl.k_end < sl.d_bulk ? sl.k_end : sl.d_bulk;
    return static_cast<int>(e - k0 < C::RAW_KT ? (e > k0 ? e - k0 : 0) : C::RAW_KT);
  };
  for (int64_t j = 0; j < sl.S && j < raw_stages; ++j)
    issue_stage<N, BF>(rows, sl, raw + j * raw_bytes, &full[j], j, warp, lane, pol, l2_hint);
  if constexpr (PRE) {
    if (sl.S > 0) {
      mbar_wait(&full[0], 0);
      centre_slice<N>(raw, rc, ring_count(sl.k_begin), warp, lane);
      named_bar(4, NT);
    }
  }
  int rs = 0, fl = 0, rn = 1;
  uint32_t ph = 0, phn = 0;
  for (int64_t j = 0; j < sl.S; ++j) {
    const int64_t k0 = sl.k_begin + j * C::RAW_KT;
    unsigned char* st = raw + rs * raw_bytes;
    if constexpr (PRE) {
      if (j + 1 < sl.S) {                          // centre the next stage before computing this one
        mbar_wait(&full[rn], phn);
        centre_slice<N>(raw + rn * raw_bytes, rc, ring_count(k0 + C::RAW_KT), warp, lane);
      }
    } else {
      mbar_wait(&full[rs], ph);
    }
    const unsigned char* rI = st + I0 * C::RAW_PITCH;
    const unsigned char* rJ = st + J0 * C::RAW_PITCH;
    const unsigned char* rC = st + rc * C::RAW_PITCH;
    if (k0 + C::RAW_KT <= sl.d_bulk) {          // a full stage, all of it in the ring
#pragma unroll 1
      for (int t = 0; t < C::PER_LANE; ++t) {
        const int k = 2 * lane + 64 * t;
        float2 vI[S], vJ[S];
#pragma unroll
        for (int a = 0; a < S; ++a) vI[a] = ld_pair<BF>(rI + a * C::RAW_PITCH, k);
#pragma unroll
        for (int b = 0; b < S; ++b) vJ[b] = ld_pair<BF>(rJ + b * C::RAW_PITCH, k);
        float hI[S], hJ[S];
        float cx = 0.f, cy = 0.f;
        if constexpr (!PRE) {
          const float2 c2 = ld_pair<BF>(rC, k);
          cx = fin(c2.x);
          cy = fin(c2.y);
        }
#pragma unroll
        for (int a = 0; a < S; ++a) hI[a] = PRE ? vI[a].x : __fsub_rn(vI[a].x, cx);
#pragma unroll
        for (int b = 0; b < S; ++b) hJ[b] = PRE ? vJ[b].x : __fsub_rn(vJ[b].x, cx);
        unit_fma<S, DIAG>(acc, hI, hJ);
#pragma unroll
        for (int a = 0; a < S; ++a) hI[a] = PRE ? vI[a].y : __fsub_rn(vI[a].y, cy);
#pragma unroll
        for (int b = 0; b < S; ++b) hJ[b] = PRE ? vJ[b].y : __fsub_rn(vJ[b].y, cy);
        unit_fma<S, DIAG>(acc, hI, hJ);
      }
    } else {                                     // the slice's last stage: ragged, tail from global
      const int cnt = static_cast<int>((sl.k_end - k0 < C::RAW_KT) ? sl.k_end - k0 : C::RAW_KT);
      using E = Elem<typename std::conditional<BF, bf2, float>::type>;
      for (int k = lane; k < cnt; k += 32) {
        const bool ring = k0 + k < sl.d_bulk;
        const bool centred = PRE && ring;         // PRE: ring values are centred already
        const float c = centred ? 0.f : fin(ring ? ld_one<BF>(rC, k) : E::value(rows.p[rc], k0 + k));
        auto h = [&](int r) {                     // padding rows: zero (their entries are never read)
          if (r >= N) return 0.f;
          const float x = ring ? ld_one<BF>(st + r * C::RAW_PITCH, k) : E::value(rows.p[r], k0 + k);
          return centred ? x : __fsub_rn(x, c);
        };
        float hI[S], hJ[S];
#pragma unroll
        for (int a = 0; a < S; ++a) hI[a] = h(I0 + a);
#pragma unroll
        for (int b = 0; b < S; ++b) hJ[b] = h(J0 + b);
        unit_fma<S, DIAG>(acc, hI, hJ);
      }
    }
    named_bar(4, NT);                             // stage j consumed (and j+1 centred) by every warp
    if (j + raw_stages < sl.S)
      issue_stage<N, BF>(rows, sl, st, &full[rs], j + raw_stages, warp, lane, pol, l2_hint);
    if (++fl == C::FLUSH_ST || j + 1 == sl.S) {
      flush<NACC>(acc, acc64, lane);
      fl = 0;
    }
    if (++rs == raw_stages) rs = 0, ph ^= 1;
    if (++rn == raw_stages) rn = 0, phn ^= 1;
  }
  const int eb = flush_base(NACC, lane);
  // wsum aliases the centre-pick scratch, free since the kernel's __syncthreads
#pragma unroll
  for (int t = 0; t < NACC / 32; ++t) wsum[warp * C::NACC_DIAG + eb + t] = acc64[t];
}

// where G_ij (i <= j < N) lives: warp and entry
template <int S>
__device__ __forceinline__ void locate(int i, int j, int* w, int* e) {
  const int gi = i / S, gj = j / S, a = i - gi * S, b = j - gj * S;
  if (gi != gj) {
    // warp of block (gi, gj): (0,1)->0 (0,2)->1 (0,3)->2 (1,2)->3 (1,3)->4 (2,3)->5
    *w = gi == 0 ? gj - 1 : gi == 1 ? gj + 1 : 5;
    *e = a * S + b;
  } else {
    const int tri = a * S - a * (a - 1) / 2 + (b - a);
    *w = (gi == 1 || gi == 2) ? 6 : 7;            // warp 6: groups 1, 2; warp 7: groups 0, 3
    *e = (gi == 2 || gi == 3) ? S * (S + 1) / 2 + tri : tri;
  }
}

template <int N, bool BF>
__global__ void __launch_bounds__(Cfg<N, BF>::THREADS, 1)
    gram_ccb_kernel(const __grid_constant__ RowPtrs rows, int64_t d, double* __restrict__ partials, int l2_hint,
                    int raw_stages, int raw_bytes) {
  using C = Cfg<N, BF>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  unsigned char* raw = base;
  unsigned char* scratch = raw + C::RAW_REGION;
  double* wsum = reinterpret_cast<double*>(scratch);
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch + C::SCRATCH);   // [RAW_STAGES_MAX]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Slice sl;
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
  // zero padding rows N..NR-1 of every slot (never written by the bulk copies)
  constexpr int PADW = (C::NR - N) * C::RAW_PITCH / 16;
  for (int s = 0; s < raw_stages; ++s)
    for (int i = threadIdx.x; i < PADW; i += C::THREADS)
      reinterpret_cast<float4*>(raw + s * raw_bytes + N * C::RAW_PITCH)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int NT = C::THREADS;
  const int rc = center_pick<NT, C::NP, BF>(rows, N, d, sl.k_begin, scratch);
  __syncthreads();                               // barriers, zero rows; the pick scratch is free again

  const int I0 = unit_gi(warp) * C::S, J0 = unit_gj(warp) * C::S;
  if (warp < 6) consume<N, BF, false>(rows, sl, raw, raw_bytes, raw_stages, full, rc, wsum, warp, lane, l2_hint, I0, J0);
  else consume<N, BF, true>(rows, sl, raw, raw_bytes, raw_stages, full, rc, wsum, warp, lane, l2_hint, I0, J0);
  named_bar(3, NT);
  double* Pm = partials + static_cast<size_t>(blockIdx.x) * N * N;
  for (int idx = threadIdx.x; idx < N * N; idx += NT) {
    int i = idx / N, jj = idx % N;
    if (i > jj) {
      const int t = i; i = jj; jj = t;
    }
    int w, e;
    locate<C::S>(i, jj, &w, &e);
    Pm[idx] = wsum[w * C::NACC_DIAG + e];
  }
}

template <int N, bool BF>
cudaError_t launch_ccb(const RowPtrs& rp, int64_t d, double* partials, int num_sms, int* n_parts,
                       cudaStream_t stream) {
  using C = Cfg<N, BF>;
  const int64_t nst = (d + C::RAW_KT - 1) / C::RAW_KT;
  int grid = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  if (nst < grid) grid = static_cast<int>(nst > 0 ? nst : 1);
  int occ = 0;
  auto kern = gram_ccb_kernel<N, BF>;
  cudaError_t e = cached_occupancy(kern, C::THREADS, C::SMEM_BYTES, &occ);
  if (e != cudaSuccess) return e;
  const int raw_bytes = C::NR * C::RAW_PITCH;
  int raw_stages = C::RAW_REGION / raw_bytes;
  if (raw_stages > C::RAW_STAGES_MAX) raw_stages = C::RAW_STAGES_MAX;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(rp, d, partials, l2_evict_first_enabled(), raw_stages,
                                                     raw_bytes);
  *n_parts = grid;
  return cudaGetLastError();
}

template <int LO, int HI, bool BF>
cudaError_t dispatch_ccb(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                         cudaStream_t stream) {
  if constexpr (LO > HI) {
    return cudaErrorInvalidValue;
  } else {
    if (n == LO) return launch_ccb<LO, BF>(rp, d, partials, num_sms, n_parts, stream);
    return dispatch_ccb<LO + 1, HI, BF>(rp, n, d, partials, num_sms, n_parts, stream);
  }
}

}  // namespace ccb
}  // namespace gar
