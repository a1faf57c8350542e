// Instantiation unit of the register-blocked CUDA-core Gram for
// kGramCcbMinN <= n <= kGramCcbMaxN (bf16 rows; gram_ccb.cuh).
#include "gram_ccb.cuh"

namespace gar {
cudaError_t launch_gram_ccb_bf16(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                             cudaStream_t stream) {
  return ccb::dispatch_ccb<kGramCcbMinN, kGramCcbMaxN, true>(rp, n, d, partials, num_sms, n_parts, stream);
}
}  // namespace gar
