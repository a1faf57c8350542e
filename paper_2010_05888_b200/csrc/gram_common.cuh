#pragma once
// gram_common.cuh — helpers of the tensor-core Gram kernel (gram_tc.cu; also
// used by the fp16-operand experiment tools/experiments/gram_f16_r2b.cu.txt):
// tcgen05 / TMEM / shared-memory-descriptor wrappers, chunk loaders and the
// per-CTA centre-row pick.  Product code for sm_100a.
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "elem.cuh"

namespace gar {
namespace gram {

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

// hi part of the tf32 split: the top 11 significant bits (exact, one LOP3).
// h - hi is then exact in fp32; the tensor core reads it as tf32 (keeping 11 of
// its <= 13 significant bits), so each product is exact to ~2^-21 relative.
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// fin(v) = v if finite else 0, branch-free (testp + selp)
__device__ __forceinline__ float fin(float v) {
  float r;
  asm("{\n\t.reg .pred p;\n\ttestp.finite.f32 p, %1;\n\tselp.f32 %0, %1, 0f00000000, p;\n\t}" : "=f"(r) : "f"(v));
  return r;
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

// 4 coordinates [k0, k0+4) of a row (k0 % 4 == 0), exactly widened to fp32,
// zero past d.
template <bool BF>
__device__ __forceinline__ float4 load_chunk_t(const float* row, int64_t k0, int64_t d) {
  if constexpr (!BF) {
    return load_chunk(row, k0, d);
  } else {
    const unsigned short* r = reinterpret_cast<const unsigned short*>(row);
    if (k0 + 4 <= d) {
      const uint2 w = __ldcs(reinterpret_cast<const uint2*>(r + k0));
      return make_float4(bf_lo(bf2{w.x}), bf_hi(bf2{w.x}), bf_lo(bf2{w.y}), bf_hi(bf2{w.y}));
    }
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k0 + 0 < d) v.x = bf16_to_f32(r[k0 + 0]);
    if (k0 + 1 < d) v.y = bf16_to_f32(r[k0 + 1]);
    if (k0 + 2 < d) v.z = bf16_to_f32(r[k0 + 2]);
    return v;
  }
}

__device__ __forceinline__ float4 widen2(uint32_t a, uint32_t b) {
  return make_float4(bf_lo(bf2{a}), bf_hi(bf2{a}), bf_lo(bf2{b}), bf_hi(bf2{b}));
}

// one 4-coordinate chunk of the raw ring, widened to fp32
template <bool BF>
__device__ __forceinline__ float4 lds_chunk(const unsigned char* a) {
  if constexpr (BF) {
    const uint2 w = *reinterpret_cast<const uint2*>(a);
    return widen2(w.x, w.y);
  } else {
    return *reinterpret_cast<const float4*>(a);
  }
}

// Byte offset of (row, 16-byte chunk c16 within a K atom) in the SW128 K-major layout.
__device__ __forceinline__ uint32_t sw128_offset(int row, int c16) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((c16 ^ (row & 7)) << 4));
}

// Centre-row pick, run by the converter warps (threads [0, NT), named barrier
// 3) while the TMA producer already streams: the most central row of a
// 128-coordinate sample of the CTA's slice, score_i = sum of the
// floor((n-1)/2) smallest sample distances D_ij.  Deterministic.  `scratch`
// (>= 49 KB of shared memory) is the idle operand ring.
// sample rows are padded by 16 bytes: the pair loop's threads read different
// rows at the same offset, conflict-free only if rows start in different banks
constexpr int kPickS = 128, kPickPitch = kPickS + 4;       // sample coordinates, row pitch (floats)
__host__ __device__ constexpr int center_pick_bytes(int np) {
  return np * kPickPitch * 4 + np * (np + 1) * 4 + np * 4;
}

template <int NT, int NP, bool BF>
__device__ int center_pick(const RowPtrs& rows, int n, int64_t d, int64_t k_begin, unsigned char* scratch) {
  constexpr int S = kPickS, SP = kPickPitch;
  float* xs = reinterpret_cast<float*>(scratch);           // [NP][SP]
  float* Ds = xs + NP * SP;                                // [NP][NP+1]
  float* score = Ds + NP * (NP + 1);                       // [NP]
  if (n <= 2) return 0;
  const int t = threadIdx.x;
  for (int e = t; e < n * (S / 4); e += NT) {
    const int r = e / (S / 4), q = e % (S / 4);
    const float4 v = load_chunk_t<BF>(rows.p[r], k_begin + 4 * q, d);
    reinterpret_cast<float4*>(xs + r * SP)[q] = make_float4(fin(v.x), fin(v.y), fin(v.z), fin(v.w));
  }
  named_bar(3, NT);
  const int np = n * (n - 1) / 2;
  for (int p = t; p < np; p += NT) {
    int i = 0, u = p;
    while (u >= n - 1 - i) { u -= n - 1 - i; ++i; }
    const int j = i + 1 + u;
    const float4* a = reinterpret_cast<const float4*>(xs + i * SP);
    const float4* b = reinterpret_cast<const float4*>(xs + j * SP);
    float acc = 0.f;
    for (int k = 0; k < S / 4; ++k) {
      const float4 x = a[k], y = b[k];
      const float dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z, dw = x.w - y.w;
      acc = fmaf(dx, dx, acc); acc = fmaf(dy, dy, acc); acc = fmaf(dz, dz, acc); acc = fmaf(dw, dw, acc);
    }
    if (!(acc <= 3.0e38f)) acc = __int_as_float(0x7f800000);
    Ds[i * (NP + 1) + j] = acc;
    Ds[j * (NP + 1) + i] = acc;
  }
  named_bar(3, NT);
  // score_i: sum (in j order) of the D_ij whose rank within row i (ties by j)
  // is below h -- the h smallest.  Ranks in parallel over (i, j) pairs.
  const int h = (n - 1) / 2;
  float* kept = xs;                                        // [NP][NP] (sample no longer needed)
  for (int e = t; e < n * n; e += NT) {
    const int i = e / n, j = e % n;
    float keep = 0.f;
    if (i != j) {
      const float v = Ds[i * (NP + 1) + j];
      int rk = 0;
      for (int k = 0; k < n; ++k) {
        const float w = Ds[i * (NP + 1) + k];
        rk += (k != i && (w < v || (w == v && k < j))) ? 1 : 0;
      }
      keep = (rk < h) ? v : 0.f;
    }
    kept[i * NP + j] = keep;
  }
  named_bar(3, NT);
  if (t < n) {
    float sc = 0.f;
    for (int j = 0; j < n; ++j) sc += kept[t * NP + j];
    score[t] = sc;
  }
  named_bar(3, NT);
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (score[i] < score[best]) best = i;
  named_bar(3, NT);                                        // scratch is reused afterwards
  return best;
}


}  // namespace gram
}  // namespace gar
