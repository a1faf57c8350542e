// coord_select.cu — host dispatch of the coordinate-selection kernel by
// (mode, rows).  Kernel body: coord_select_impl.cuh; instantiations are split
// over coord_inst_*.cu so they compile in parallel.
#include "coord_select_impl.cuh"

namespace gar {

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

cudaError_t launch_coord_select(int mode, const CoordLaunch& L, cudaStream_t stream) {
  if (L.d == 0) return cudaSuccess;
  if (L.R < 1 || L.R > GAR_MAX_N) return cudaErrorInvalidValue;
  if (mode == kModeAverage) {
    if (L.R == 1) return launch_copy_row(L, stream);
    return launch_mode<kModeAverage, 0>(L, stream);
  }
  const int band = (L.R - 1) / 16;
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
