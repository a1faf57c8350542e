// GENERATED instantiation unit (split for parallel compilation).
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_bulyan_49_64(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_range<kModeBulyan, 49, 64, float>(L, stream);
}
}  // namespace gar
