// gram.h — internal launch interface: Gram partials, their reduction, and the
// selection kernel (rows a5-a7 of DESIGN.md §1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gar {

// Upper bound on the number of per-CTA partial Gram matrices (>= SM count).
constexpr int kGramMaxParts = 160;

// Per-coordinate centring reference c_k (DESIGN.md §4 "Gram"): c_k =
// fin(x_{r*,k}) (fin(v) = v if finite else 0), where r* is the most central
// row of a 128-coordinate sample of the CTA's slice (gram_tc.cu center_pick:
// smallest sum of the floor((n-1)/2) smallest sample distances).  Each CTA
// picks its own r*; a per-coordinate translation leaves D_ij unchanged
// mathematically.

// Partial Gram matrices of the centred rows, one fp64 [n x n] per CTA,
// written to partials[p*n*n ...].  *n_parts receives the number written.
// stage_rows (optional, n device pointers): every row's [0, d) is also copied
// there from the kernel's staging ring (fused ingress staging).
cudaError_t launch_gram_partials(const float* const* rows, int n, int64_t d, double* partials,
                                 int num_sms, int* n_parts, cudaStream_t stream,
                                 float* const* stage_rows = nullptr, int dtype = 0 /* ElemType */);

// The same contract on the CUDA cores (fp32 FFMA, all n(n+1)/2 products per
// lane, fp64 across stages; gram_cc.cu) for n <= kGramCcMaxN; launch_gram_partials
// uses it there.
constexpr int kGramCcMaxN = 15;
cudaError_t launch_gram_cc(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                           int* n_parts, cudaStream_t stream, int dtype);
// ... and for kGramCcMaxN < n <= kGramCckLimit with the pair triangle cut into
// two chunks over warps (gram_cck.cu); launch_gram_partials uses it up to
// kGramCckMaxN.
constexpr int kGramCckLimit = 24;
constexpr int kGramCckMaxN = 24;
// ... and register-blocked over 8 warps (4 row groups of S = 9: 6 block units,
// 2 triangle-pair units; gram_ccb.cuh) for kGramCcbMinN <= n <= kGramCcbMaxN,
// where it beats the NP = 64 tensor-core pass (1.05 vs 1.27 ms at n = 35)
constexpr int kGramCcbMinN = 33;
constexpr int kGramCcbMaxN = 36;
cudaError_t launch_gram_cck(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                            int* n_parts, cudaStream_t stream, int dtype);

// G = sum_p partials[p] in fixed order p = 0..n_parts-1 (deterministic).
cudaError_t launch_gram_reduce(const double* partials, int n_parts, int n, double* G,
                               cudaStream_t stream);

enum SelectRule { kSelDistancesOnly = 0, kSelMultiKrum = 1, kSelBulyan = 2 };

// From G: D (fp64 n x n, optional), then the selection of `rule`:
// Multi-Krum -> m indices by ascending (score, index); Bulyan -> n-2f indices in
// round order.  idx_out: device int32.
cudaError_t launch_select(const double* G, int n, int f, int m, int rule, int32_t* idx_out,
                          double* D_out, cudaStream_t stream);

// Peer-memory Gram exchange (exchange.cu): slot arrays double[world][n*n]
// and flag arrays uint32[world] of every rank, as mapped on this GPU.
constexpr int kMaxWorld = 8;
struct PeerSlots {
  double* p[kMaxWorld];
};
struct PeerFlags {
  uint32_t* p[kMaxWorld];
};
cudaError_t launch_gram_exchange(const double* partials, int n_parts, int n, const PeerSlots& slots,
                                 const PeerFlags& flags, int world, int rank, uint32_t epoch, double* G,
                                 cudaStream_t stream);

// MDA selection (mda.cu): scratch of mda_workspace_bytes(n) bytes, at most
// kMdaMaxCtas enumeration CTAs; idx_out = the n - f kept indices, ascending.
constexpr int kMdaMaxCtas = 1024;
size_t mda_workspace_bytes(int n);
cudaError_t launch_mda_select(const double* D, int n, int f, void* scratch, int num_sms, int32_t* idx_out,
                              cudaStream_t stream);

// Rows with a non-finite value (membership.cu; SPEC's vector-level sanitize).
cudaError_t launch_nonfinite_rows(const float* const* rows, int n, int64_t d, uint64_t* mask, int num_sms,
                                  cudaStream_t stream);

// Trimmed-set membership masks (membership.cu; verification entry point).
cudaError_t launch_trimmed_membership(const float* const* rows, int n, int f, int64_t d, uint64_t* mask,
                                      int num_sms, cudaStream_t stream);

}  // namespace gar
