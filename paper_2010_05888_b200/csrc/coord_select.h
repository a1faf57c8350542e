// coord_select.h — internal launch interface of the coordinate-selection kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace gar {

enum CoordMode { kModeAverage = 0, kModeMedian = 1, kModeTrimmed = 2, kModeBulyan = 3 };

struct CoordLaunch {
  const float* const* rows;   // host array of n device row pointers (bf16 rows: type-punned)
  int n;                      // number of input rows
  const int32_t* idx;         // device: R selected indices (any order) or nullptr
  int R;                      // rows consumed per coordinate (n, m or theta)
  int f;                      // trim per side / Bulyan f
  int64_t d;                  // coordinates
  float* out;                 // device fp32[d]
  OutPtrs extra;              // further destinations (n = 0: none)
  int num_sms;
  int dtype;                  // ElemType (elem.cuh): kF32 or kBF16
};

cudaError_t launch_coord_select(int mode, const CoordLaunch& L, cudaStream_t stream);

// Tuning knob: L2 evict-first policy on the streaming bulk copies (default off:
// measured no gain; GAR_L2_EVICT_FIRST=1 enables it).  Read once per process.
int l2_evict_first_enabled();

}  // namespace gar
