// GENERATED instantiation unit (split for parallel compilation): bf16 rows.
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_bulyan_17_32_bf16(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_range<kModeBulyan, 17, 32, bf2>(L, stream);
}
}  // namespace gar
