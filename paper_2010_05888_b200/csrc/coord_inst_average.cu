// Instantiation unit of the direct-load Average with a compile-time row count
// for R <= 8, so every row's load is issued before the fp64 sum in index
// order.  Measured (profiles/r1_sweep_C5.md notes): n = 7 0.171 -> 0.140 ms;
// at n = 11, 15 and 63 the compile-time form was 4-10 % slower than the
// runtime-R loop, which those sizes keep.
#include "coord_select_impl.cuh"
namespace gar {
template <int LO, int HI>
inline cudaError_t dispatch_avg(const CoordLaunch& L, cudaStream_t stream) {
  if constexpr (LO > HI) {
    return launch_ldg<kModeAverage, 0>(L, stream);
  } else {
    if (L.R == LO) return launch_ldg<kModeAverage, LO>(L, stream);
    return dispatch_avg<LO + 1, HI>(L, stream);
  }
}

cudaError_t launch_coord_average_ldg(const CoordLaunch& L, cudaStream_t stream) {
  return dispatch_avg<2, 8>(L, stream);
}
}  // namespace gar
