// GENERATED instantiation unit (split for parallel compilation).
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_median_1_16(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_range<kModeMedian, 1, 16, float>(L, stream);
}
}  // namespace gar
