// coord_select.cu — host dispatch of the coordinate-selection kernel by
// (mode, rows).  Kernel body: coord_select_impl.cuh; instantiations are split
// over coord_inst_*.cu so they compile in parallel.
#include <cstdlib>

#include "coord_select_impl.cuh"

namespace gar {

// Krum combine (one selected row): out = fp32((0 + x) / 1) = x + 0 (-0 -> +0),
// a plain vectorised streaming copy.
__global__ void __launch_bounds__(256) copy_row_kernel(const __grid_constant__ RowPtrs rows, const int32_t* idx,
                                                        float* __restrict__ out, const __grid_constant__ OutPtrs extra,
                                                        int64_t d) {
  const float* src = rows.p[idx ? idx[0] : 0];
  const int64_t n4 = d >> 2;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n4; q += int64_t(gridDim.x) * blockDim.x) {
    float4 v = __ldcs(reinterpret_cast<const float4*>(src) + q);
    v.x = __fadd_rn(v.x, 0.0f); v.y = __fadd_rn(v.y, 0.0f); v.z = __fadd_rn(v.z, 0.0f); v.w = __fadd_rn(v.w, 0.0f);
    if (extra.sgd) {
      float4 w = __ldcs(reinterpret_cast<const float4*>(out) + q);
      w.x = fmaf(-extra.lr, v.x, w.x); w.y = fmaf(-extra.lr, v.y, w.y);
      w.z = fmaf(-extra.lr, v.z, w.z); w.w = fmaf(-extra.lr, v.w, w.w);
      __stcs(reinterpret_cast<float4*>(out) + q, w);
      continue;
    }
    if (extra.mc) {
      mc_store4(extra.mc + 4 * q, v);
      continue;
    }
    __stcs(reinterpret_cast<float4*>(out) + q, v);
    for (int j = 0; j < extra.n; ++j) reinterpret_cast<float4*>(extra.p[j])[q] = v;
  }
  const int64_t k = (n4 << 2) + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (blockIdx.x == 0 && k < d) store_result(out, extra, k, __fadd_rn(src[k], 0.0f));
}

// The same copy from a bf16 row: out = fp32(x) + 0 (exact widening, R16).
__global__ void __launch_bounds__(256) copy_row_bf16_kernel(const __grid_constant__ RowPtrs rows, const int32_t* idx,
                                                             float* __restrict__ out,
                                                             const __grid_constant__ OutPtrs extra, int64_t d) {
  const unsigned short* src = reinterpret_cast<const unsigned short*>(rows.p[idx ? idx[0] : 0]);
  const int64_t n8 = d >> 3;                      // 16-byte chunks of 8 bf16
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < n8; q += int64_t(gridDim.x) * blockDim.x) {
    const uint4 w = __ldcs(reinterpret_cast<const uint4*>(src) + q);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
    float v[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[2 * j] = __fadd_rn(bf_lo(bf2{u[j]}), 0.0f);
      v[2 * j + 1] = __fadd_rn(bf_hi(bf2{u[j]}), 0.0f);
    }
    float4* o = reinterpret_cast<float4*>(out) + 2 * q;
    if (extra.sgd) {
      float4 a = __ldcs(o), b = __ldcs(o + 1);
      a.x = fmaf(-extra.lr, v[0], a.x); a.y = fmaf(-extra.lr, v[1], a.y);
      a.z = fmaf(-extra.lr, v[2], a.z); a.w = fmaf(-extra.lr, v[3], a.w);
      b.x = fmaf(-extra.lr, v[4], b.x); b.y = fmaf(-extra.lr, v[5], b.y);
      b.z = fmaf(-extra.lr, v[6], b.z); b.w = fmaf(-extra.lr, v[7], b.w);
      __stcs(o, a);
      __stcs(o + 1, b);
      continue;
    }
    const float4 a = make_float4(v[0], v[1], v[2], v[3]), b = make_float4(v[4], v[5], v[6], v[7]);
    if (extra.mc) {
      mc_store4(extra.mc + 8 * q, a);
      mc_store4(extra.mc + 8 * q + 4, b);
      continue;
    }
    __stcs(o, a);
    __stcs(o + 1, b);
    for (int j = 0; j < extra.n; ++j) {
      reinterpret_cast<float4*>(extra.p[j])[2 * q] = a;
      reinterpret_cast<float4*>(extra.p[j])[2 * q + 1] = b;
    }
  }
  const int64_t k = (n8 << 3) + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (blockIdx.x == 0 && k < d) store_result(out, extra, k, __fadd_rn(bf16_to_f32(src[k]), 0.0f));
}

int l2_evict_first_enabled() {
  static const int v = [] {
    const char* e = getenv("GAR_L2_EVICT_FIRST");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v;
}

int coord_loader_ldg(int mode, int R) {
  static const int forced = [] {
    const char* e = getenv("GAR_COORD_LOADER");
    if (e && e[0] == 'l') return 1;
    if (e && e[0] == 't') return 0;
    return -1;
  }();
  if (forced >= 0) return forced;
  // Measured per mode on B200 across n = 7..63 (profiles/r1_loader_choice.md):
  // the TMA ring wins for the Median at every row count, for averages at 17..32
  // and 48..64 rows, for the trimmed mean above 12 rows, and for the Bulyan
  // phase (24 consumer warps) at 17..32 rows; direct loads win elsewhere.
  switch (mode) {
    case kModeMedian: return 0;
    case kModeAverage: return ((R > 16 && R <= 32) || R >= 48) ? 0 : 1;
    case kModeTrimmed: return R > 12 ? 0 : 1;
    case kModeBulyan: return (R > 16 && R <= 32) ? 0 : 1;
    default: return 1;
  }
}

inline cudaError_t launch_copy_row(const CoordLaunch& L, cudaStream_t stream) {
  RowPtrs rp;
  for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < L.n) ? L.rows[i] : nullptr;
  const int per = (L.dtype == kBF16) ? 8 : 4;     // coordinates per thread-iteration
  int64_t blocks = (L.d / per + 255) / 256;
  const int64_t cap = int64_t(L.num_sms) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (L.dtype == kBF16)
    copy_row_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(rp, L.idx, L.out, L.extra, L.d);
  else
    copy_row_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(rp, L.idx, L.out, L.extra, L.d);
  return cudaGetLastError();
}

cudaError_t launch_coord_median_1_16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_17_32(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_33_48(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_49_64(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_1_16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_17_32(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_33_48(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_49_64(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_1_16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_17_32(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_33_48(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_49_64(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_average_ldg(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_1_16_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_17_32_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_33_48_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_median_49_64_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_1_16_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_17_32_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_33_48_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_trimmed_49_64_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_1_16_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_17_32_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_33_48_bf16(const CoordLaunch& L, cudaStream_t stream);
cudaError_t launch_coord_bulyan_49_64_bf16(const CoordLaunch& L, cudaStream_t stream);

// A/B knob: GAR_AVG_RUNTIME_R=1 keeps the runtime-row-count direct-load Average
static int getenv_flag_avg_runtime() {
  static const int v = getenv("GAR_AVG_RUNTIME_R") != nullptr ? 1 : 0;
  return v;
}

cudaError_t launch_coord_select(int mode, const CoordLaunch& L, cudaStream_t stream) {
  if (L.d == 0) return cudaSuccess;
  if (L.R < 1 || L.R > GAR_MAX_N) return cudaErrorInvalidValue;
  if (L.dtype != kF32 && L.dtype != kBF16) return cudaErrorInvalidValue;
  if (mode == kModeAverage) {
    if (L.R == 1) return launch_copy_row(L, stream);
    if (L.dtype == kBF16) return launch_mode<kModeAverage, 0, bf2>(L, stream);
    if (L.R <= 8 && coord_loader_ldg(kModeAverage, L.R) && getenv_flag_avg_runtime() == 0) return launch_coord_average_ldg(L, stream);
    return launch_mode<kModeAverage, 0, float>(L, stream);
  }
  const int band = (L.R - 1) / 16;
  if (L.dtype == kBF16) {
    switch (mode) {
      case kModeMedian:
        switch (band) { case 0: return launch_coord_median_1_16_bf16(L, stream); case 1: return launch_coord_median_17_32_bf16(L, stream); case 2: return launch_coord_median_33_48_bf16(L, stream); case 3: return launch_coord_median_49_64_bf16(L, stream); }
        break;
      case kModeTrimmed:
        switch (band) { case 0: return launch_coord_trimmed_1_16_bf16(L, stream); case 1: return launch_coord_trimmed_17_32_bf16(L, stream); case 2: return launch_coord_trimmed_33_48_bf16(L, stream); case 3: return launch_coord_trimmed_49_64_bf16(L, stream); }
        break;
      case kModeBulyan:
        switch (band) { case 0: return launch_coord_bulyan_1_16_bf16(L, stream); case 1: return launch_coord_bulyan_17_32_bf16(L, stream); case 2: return launch_coord_bulyan_33_48_bf16(L, stream); case 3: return launch_coord_bulyan_49_64_bf16(L, stream); }
        break;
      default: break;
    }
    return cudaErrorInvalidValue;
  }
  switch (mode) {
    case kModeMedian:
      switch (band) { case 0: return launch_coord_median_1_16(L, stream); case 1: return launch_coord_median_17_32(L, stream); case 2: return launch_coord_median_33_48(L, stream); case 3: return launch_coord_median_49_64(L, stream); }
      break;
    case kModeTrimmed:
      switch (band) { case 0: return launch_coord_trimmed_1_16(L, stream); case 1: return launch_coord_trimmed_17_32(L, stream); case 2: return launch_coord_trimmed_33_48(L, stream); case 3: return launch_coord_trimmed_49_64(L, stream); }
      break;
    case kModeBulyan:
      switch (band) { case 0: return launch_coord_bulyan_1_16(L, stream); case 1: return launch_coord_bulyan_17_32(L, stream); case 2: return launch_coord_bulyan_33_48(L, stream); case 3: return launch_coord_bulyan_49_64(L, stream); }
      break;
    default: break;
  }
  return cudaErrorInvalidValue;
}

}  // namespace gar
