// gram_tc.cu — product Gram partials.  (Temporary: forwards to the SIMT
// reference kernel until the tcgen05 kernel lands.)
#include "gram.h"

namespace gar {

cudaError_t launch_gram_partials(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                                 int* n_parts, cudaStream_t stream) {
  return launch_gram_partials_simt(rows, n, d, partials, num_sms, n_parts, stream);
}

}  // namespace gar
