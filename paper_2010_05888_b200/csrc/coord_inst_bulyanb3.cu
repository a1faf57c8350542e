// Instantiation unit of the beta = 3 Bulyan phase: theta = 2f + 3 with
// n = 4f + 3 <= 64 gives theta in {5, 7, ..., 33}.
#include "coord_select_impl.cuh"
namespace gar {
cudaError_t launch_coord_bulyanb3(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_b3<5, 33>(L, stream);
}
}  // namespace gar
