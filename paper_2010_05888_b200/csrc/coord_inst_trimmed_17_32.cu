// GENERATED instantiation unit (split for parallel compilation).
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_trimmed_17_32(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_range<kModeTrimmed, 17, 32, float>(L, stream);
}
}  // namespace gar
