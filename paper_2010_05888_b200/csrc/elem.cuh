#pragma once
// elem.cuh — element types of the gradient rows (product code, sm_100a).
//
// fp32 rows are processed one coordinate per thread as `float`.  bf16 rows
// (R16: every bf16 value is widened EXACTLY to fp32
// and the rules are the fp32 definitions on the widened values) are processed
// two adjacent coordinates per thread as `bf2`: one 32-bit register holding
// the bf16 values of coordinates 2j (low half) and 2j+1 (high half), so the
// order-statistic networks run on packed min.bf16x2 / max.NaN.bf16x2, one
// instruction per compare for two coordinates.  bf16 orders exactly like its
// fp32 widening (same sign / exponent / leading mantissa bits), so a network
// over bf2 sorts each half exactly as the fp32 network sorts the widened
// values; the NaN semantics of the pair (min drops a NaN operand, max.NaN
// propagates it) are those of the fp32 pair, so a NaN moves like +inf (R1).
#include <cstdint>
#include <cuda_runtime.h>

namespace gar {

enum ElemType { kF32 = 0, kBF16 = 1 };

struct bf2 {
  uint32_t u;
};

// exact widening of the halves
__device__ __forceinline__ float bf_lo(bf2 x) { return __uint_as_float(x.u << 16); }
__device__ __forceinline__ float bf_hi(bf2 x) { return __uint_as_float(x.u & 0xFFFF0000u); }
__device__ __forceinline__ float bf_half(bf2 x, int h) { return h ? bf_hi(x) : bf_lo(x); }
__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }

// compare-exchange primitives of the networks (networks.cuh)
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float vmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ bf2 vmin(bf2 a, bf2 b) {
  bf2 r;
  asm("min.bf16x2 %0, %1, %2;" : "=r"(r.u) : "r"(a.u), "r"(b.u));
  return r;
}
__device__ __forceinline__ bf2 vmax_nan(bf2 a, bf2 b) {
  bf2 r;
  asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r.u) : "r"(a.u), "r"(b.u));
  return r;
}

// Per element type: coordinates per thread-element (EPT), bytes per
// coordinate (ES), and the exact fp32 value of coordinate k of a row (for the
// rare direct reads: ragged tails, Bulyan's exact tie path).
template <class T>
struct Elem;
template <>
struct Elem<float> {
  static constexpr int EPT = 1, ES = 4;
  static __device__ __forceinline__ float value(const void* row, int64_t k) {
    return __ldg(static_cast<const float*>(row) + k);
  }
};
template <>
struct Elem<bf2> {
  static constexpr int EPT = 2, ES = 2;
  static __device__ __forceinline__ float value(const void* row, int64_t k) {
    return bf16_to_f32(__ldg(static_cast<const unsigned short*>(row) + k));
  }
};

}  // namespace gar
