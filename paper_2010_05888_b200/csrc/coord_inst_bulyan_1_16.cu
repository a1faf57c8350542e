// GENERATED instantiation unit (split for parallel compilation).
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_bulyan_1_16(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_range<kModeBulyan, 1, 16, float>(L, stream);
}
}  // namespace gar
