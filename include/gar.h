/* gar.h — libgar: the C-ABI boundary of the Garfield GAR hot path on B200.
 *
 * Garfield (arXiv 2010.05888) §3.3 "Statistically Robust GARs" (PAPER.md
 * l.198-225): "A GAR is merely a function of (R^d)^q -> R^d ... these GARs wait
 * for q vectors before applying some functions on them" (l.201-203).  The
 * paper's aggregation module exposes two calls, init(name, n, f) and
 * aggregate(n tensors), the device being chosen by where the inputs live
 * (§4.1 "Aggregation").  libgar is that module for
 * B200 (sm_100a) GPUs; every step runs in hand-written CUDA kernels.
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - grads:  HOST array of n DEVICE pointers; grads[i] is worker i's gradient,
 *            fp32[d] (or fp32[d_local] for the sharded calls), 16-byte
 *            aligned.  The array itself is copied into kernel parameters at
 *            call time; the caller may free it when the call returns.
 *  - 1 <= n <= GAR_MAX_N (64), f >= 0, d >= 0.
 *  - out:    DEVICE fp32[d], 16-byte aligned, must not alias any grads[i].
 *  - indices_dev: DEVICE int32 array of at least GAR_MAX_N entries.
 *  - stream: the CUDA stream all work is enqueued on (NULL = legacy default).
 *  - Ownership: the caller owns every buffer; libgar never allocates device
 *    memory except in gar_aggregate (7-argument convenience form), which
 *    takes its workspace from cudaMallocAsync on `stream`.
 *  - Argument checks run synchronously before any launch; on failure nothing
 *    is written.  Execution is asynchronous: results are valid once `stream`
 *    reaches the point of the call.  Launch failures return GAR_ERR_CUDA.
 *  - No CPU fallback: host pointers in grads/out -> GAR_ERR_INVALID_ARGUMENT.
 *  - Stateless and re-entrant; concurrent calls need separate workspaces.
 *  - Results are bitwise deterministic for fixed inputs.
 *
 * Numerics (DESIGN.md §3 readings R1-R14): order statistics on canonical
 * values (NaN -> +inf, -0 -> +0), averages as fp64 sums rounded once to fp32,
 * squared Euclidean distances from a tensor-core Gram matrix, ties to the
 * lower input index.
 */
#ifndef GARFIELD_B200_GAR_H_
#define GARFIELD_B200_GAR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gar_stream_t; /* == cudaStream_t */

#define GAR_MAX_N 64

typedef enum {
  GAR_AVERAGE = 0,      /* PAPER.md l.146-152 (§2.2), control rule l.553-554          */
  GAR_MEDIAN = 1,       /* coordinate-wise median, q >= 2f+1, l.207-208              */
  GAR_TRIMMED_MEAN = 2, /* coordinate-wise trimmed mean, l.316 footnote; R6          */
  GAR_KRUM = 3,         /* Multi-Krum with m = 1, l.210-212; R10                     */
  GAR_MULTI_KRUM = 4,   /* average of the m smallest-score inputs, l.210-212         */
  GAR_BULYAN = 5,       /* iterated Krum + coordinate phase, l.219-225; R7, R8       */
  GAR_MDA = 6,          /* minimum-diameter averaging, l.214-217; R13; q >= 2f+1,   */
                        /* C(q, f) <= 2^31 (GAR_ERR_UNSUPPORTED above)              */
  GAR_MEAN_AROUND_MEDIAN = 7 /* per coordinate, mean of the n-2f values closest to   */
                        /* the median, l.316 fn.; R14; q >= 2f+1                    */
} gar_rule;

typedef enum {
  GAR_OK = 0,
  GAR_ERR_INVALID_ARGUMENT = 1, /* null/host pointer, n outside [1,64], f<0, d<0, out aliases an input, bad rule */
  GAR_ERR_QUORUM = 2,           /* n < 2f+1 (median, trimmed, MDA, mean around median) | 2f+3 (Krum family) | 4f+3 (Bulyan); l.208, l.212, l.217, l.225 */
  GAR_ERR_INVALID_M = 3,        /* Multi-Krum m outside [1, n-f-2] (l.210)                              */
  GAR_ERR_ALIGNMENT = 4,        /* a row or out pointer not 16-byte aligned                             */
  GAR_ERR_UNSUPPORTED = 5,      /* selection asked of a coordinate-wise rule; MDA beyond its budget    */
  GAR_ERR_WORKSPACE = 6,        /* workspace missing or smaller than gar_workspace_bytes()             */
  GAR_ERR_CUDA = 7              /* a CUDA call or kernel launch failed                                  */
} gar_status;

/* Human-readable name of a status code (static storage). */
const char* gar_status_string(gar_status s);

/* Description of the last CUDA failure (GAR_ERR_CUDA) seen by the calling
 * thread inside libgar: cudaGetErrorString text and code; "" if none. */
const char* gar_last_error(void);

/* Bytes of device workspace gar_aggregate_ex / gar_select / gar_gram_partial
 * need for (rule, n, f, d); 0 for the coordinate-wise rules.  Pure host
 * function (no CUDA call).  Returns 0 on invalid arguments. */
size_t gar_workspace_bytes(gar_rule rule, int n, int f, int64_t d);

/* Number of indices the selection of (rule, n, f, m) produces: Krum 1,
 * Multi-Krum m (0 -> n-f-2), Bulyan n-2f; 0 for coordinate-wise rules or on
 * invalid arguments.  Pure host function. */
int gar_num_selected(gar_rule rule, int n, int f, int m);

/* The argument checks every entry point runs first, as a pure host function
 * (no CUDA call): GAR_OK, GAR_ERR_INVALID_ARGUMENT (unknown rule, n outside
 * [1, 64], f < 0), GAR_ERR_QUORUM (n below the rule's bound: PAPER.md l.208,
 * l.212, l.225), GAR_ERR_INVALID_M (Multi-Krum m outside [1, n-f-2], l.210)
 * or GAR_ERR_UNSUPPORTED (MDA with more than 2^31 candidate subsets C(n, f)).
 * Lets a binding report the real reason where gar_num_selected returns 0. */
gar_status gar_check_args(gar_rule rule, int n, int f, int m);

/* out = GAR_rule(grads[0..n)) over d coordinates (default m = n-f-2 for
 * Multi-Krum).  Allocates its workspace with cudaMallocAsync on `stream`. */
gar_status gar_aggregate(gar_rule rule, const float* const* grads, int n, int f, int64_t d,
                         float* out, gar_stream_t stream);

/* Full form.  m: Multi-Krum selection size (0 -> n-f-2; ignored by other
 * rules).  indices_dev: optional DEVICE int32[>= n_selected] receiving the
 * selected input indices in selection order (Krum family; may be NULL).
 * workspace: DEVICE buffer of >= gar_workspace_bytes(rule, n, f, d) bytes
 * (may be NULL for the coordinate-wise rules). */
gar_status gar_aggregate_ex(gar_rule rule, const float* const* grads, int n, int f, int m,
                            int64_t d, float* out, int32_t* indices_dev, void* workspace,
                            size_t workspace_bytes, gar_stream_t stream);

/* Selection only (Krum, Multi-Krum, Bulyan, MDA): indices in selection order
 * — ascending (score, index) for Krum/Multi-Krum, round order for Bulyan,
 * ascending index for MDA's minimum-diameter subset of n - f — into
 * indices_dev.  *n_selected_host (optional) receives the count, known
 * without synchronising. */
gar_status gar_select(gar_rule rule, const float* const* grads, int n, int f, int m, int64_t d,
                      int32_t* indices_dev, int* n_selected_host, void* workspace,
                      size_t workspace_bytes, gar_stream_t stream);

/* Pairwise squared distances D (DEVICE fp64[n*n], row-major, symmetric,
 * zero diagonal, non-finite -> +inf) from the tensor-core Gram matrix:
 * D_ij = G_ii + G_jj - 2 G_ij with G the Gram matrix of the centred rows
 * (row a5).  workspace as for Krum. */
gar_status gar_distances(const float* const* grads, int n, int64_t d, double* D_dev,
                         void* workspace, size_t workspace_bytes, gar_stream_t stream);

/* ---- d-sharded building blocks (multi-GPU) -----------------
 * A rank holding coordinates [lo, lo+d_local) of every gradient calls
 * gar_gram_partial, sums gram_dev over ranks (NCCL all-reduce, fp64), then
 * gar_select_from_gram (identical on every rank) and gar_combine on its slice.
 * The centring reference of the Gram is per-coordinate, so partial Grams of
 * disjoint coordinate slices add up to the Gram of the whole vectors. */

/* gram_dev: DEVICE fp64[n*n], the Gram matrix of the centred local slice. */
gar_status gar_gram_partial(const float* const* grads, int n, int64_t d_local, double* gram_dev,
                            void* workspace, size_t workspace_bytes, gar_stream_t stream);

/* Selection from a (summed) Gram matrix; same outputs as gar_select.
 * workspace: >= gar_workspace_bytes(rule, n, f, 0) bytes (required for MDA,
 * unused by the others). */
gar_status gar_select_from_gram(gar_rule rule, const double* gram_dev, int n, int f, int m,
                                int32_t* indices_dev, int* n_selected_host, void* workspace,
                                size_t workspace_bytes, gar_stream_t stream);

/* Combine step on a coordinate slice given the selection: Krum copies the
 * selected row, Multi-Krum averages the m selected rows, MDA the n-f selected
 * rows (fp64, index order), Bulyan runs its coordinate phase over the n-2f
 * selected rows.  indices_dev as produced by
 * gar_select / gar_select_from_gram. */
gar_status gar_combine(gar_rule rule, const float* const* grads, int n, int f, int m,
                       int64_t d_local, const int32_t* indices_dev, float* out,
                       gar_stream_t stream);

/* ---- fused output all-gather (multi-GPU) ----------------------
 * As gar_aggregate_ex / gar_combine, but every result coordinate is ALSO
 * stored at extra_outs[j][i] (j < n_extra <= 8) by the producing kernel itself.
 * For a d-sharded rank, extra_outs[j] is the position of this rank's slice in
 * GPU j's replicated output buffer, mapped into this GPU's address space
 * (e.g. torch symmetric memory): the all-gather of the aggregate then travels
 * over NVLink inside the kernel that computes it instead of in a separate
 * collective.  The caller synchronises the ranks before reading (barrier).
 * extra_outs: host array of device or peer-mapped pointers, 16-byte aligned,
 * not aliasing the inputs; they are not checked for host memory. */
gar_status gar_aggregate_bcast(gar_rule rule, const float* const* grads, int n, int f, int m,
                               int64_t d, float* out, float* const* extra_outs, int n_extra,
                               int32_t* indices_dev, void* workspace, size_t workspace_bytes,
                               gar_stream_t stream);

gar_status gar_combine_bcast(gar_rule rule, const float* const* grads, int n, int f, int m,
                             int64_t d_local, const int32_t* indices_dev, float* out,
                             float* const* extra_outs, int n_extra, gar_stream_t stream);

/* gar_aggregate_mcast / gar_combine_mcast: gar_aggregate_ex / gar_combine
 * with the result written through a MULTICAST address instead (the d-sharded
 * output all-gather the north_star names, done by the
 * producing kernel over NVLink SHARP): out_mc is the multicast virtual
 * address (e.g. torch symmetric memory's multicast_ptr + byte offset) of the
 * region whose local mapping is `out`; each result is stored once with
 * multimem.st and the NVSwitch writes it into every member GPU's buffer,
 * `out` included, so nothing is stored to `out` directly.  out_mc: non-null,
 * 16-byte aligned (GAR_ERR_INVALID_ARGUMENT / GAR_ERR_ALIGNMENT), not checked
 * with cudaPointerGetAttributes.  Visibility on the other GPUs needs the
 * caller's cross-GPU barrier after the call, as for the _bcast variants. */
gar_status gar_aggregate_mcast(gar_rule rule, const float* const* grads, int n, int f, int m,
                               int64_t d, float* out, float* out_mc, int32_t* indices_dev,
                               void* workspace, size_t workspace_bytes, gar_stream_t stream);

gar_status gar_combine_mcast(gar_rule rule, const float* const* grads, int n, int f, int m,
                             int64_t d_local, const int32_t* indices_dev, float* out, float* out_mc,
                             gar_stream_t stream);

/* Fused server step (the update on the far side of the path, PAPER.md
 * l.122-125, x <- x - gamma * GAR(gradients)):
 * params[k] <- fma(-lr, GAR(grads)[k], params[k]) with one rounding, applied
 * by the producing kernel instead of storing the aggregate (saves the
 * aggregate's write and re-read).  params: DEVICE fp32[d], 16-byte aligned,
 * in/out, not aliasing the inputs; lr finite.  Otherwise as
 * gar_aggregate_ex / gar_combine; d-sharded callers pass their parameter
 * slice (the ZeRO-style consumer of the sharded output). */
gar_status gar_aggregate_sgd(gar_rule rule, const float* const* grads, int n, int f, int m,
                             int64_t d, float* params, float lr, int32_t* indices_dev,
                             void* workspace, size_t workspace_bytes, gar_stream_t stream);

gar_status gar_combine_sgd(gar_rule rule, const float* const* grads, int n, int f, int m,
                           int64_t d_local, const int32_t* indices_dev, float* params, float lr,
                           gar_stream_t stream);

/* d-sharded Gram exchange without a collective library (row a10, PAPER.md
 * l.437-438): the Gram partial of this rank's slice (as gar_gram_partial),
 * stored into slot `rank` of every rank's slot array over NVLink, then a
 * flag handshake, then gram_dev = the sum of the `world` slots in rank order
 * — the whole-vector Gram matrix, bit-identical on every rank.
 * peer_slots: host array [world] of the slot arrays (DEVICE fp64
 *   [world][n*n], 8-byte aligned) of every rank as mapped on this GPU (e.g.
 *   torch symmetric memory); the caller alternates two slot arrays between
 *   consecutive calls (a rank may run one call ahead of another).
 * peer_flags: host array [world] of every rank's flag array (uint32[world],
 *   zero before the first call, 4-byte aligned).
 * epoch: > the previous call's epoch, the same on every rank for one call.
 * world <= 8.  A rank that does not arrive within ~10 s makes the kernel
 * trap instead of hanging: the stream's context then holds a sticky launch
 * error, which this or the next call (or a stream synchronize) reports
 * (GAR_ERR_CUDA); no result is produced.  workspace as for gar_gram_partial.
 * stage_rows (optional, host array of n DEVICE fp32[d_local] buffers,
 * 16-byte aligned): the Gram kernel also writes every row's slice there from
 * its staging ring (bulk stores), so rows read from other GPUs' memory
 * (worker-major ingress) land locally for the combine step
 * while the Gram is computed; NULL to skip. */
gar_status gar_gram_exchange(const float* const* grads, int n, int64_t d_local,
                             double* const* peer_slots, uint32_t* const* peer_flags, int rank,
                             int world, uint32_t epoch, double* gram_dev, float* const* stage_rows,
                             void* workspace, size_t workspace_bytes, gar_stream_t stream);

/* Non-finite rows (the vector-level sanitize that counts
 * non-finite payloads toward f): *mask_dev (DEVICE uint64,
 * 8-byte aligned) <- bit i set iff row i holds a NaN or +-inf in [0, d).
 * Reads every input once.  The caller drops those rows and aggregates the
 * rest with f reduced by their count (paper_2010_05888_b200.sanitize). */
gar_status gar_nonfinite_rows(const float* const* grads, int n, int64_t d, uint64_t* mask_dev,
                              gar_stream_t stream);

/* Trimmed-set membership (verification entry point for row a3, PAPER.md
 * l.316 footnote; the north_star's bit-exact "trimmed-set membership"): bit i
 * of mask_dev[k] is set iff input i is among the n - 2f values the trimmed
 * mean keeps at coordinate k — canonical order (NaN -> +inf, -0 -> +0), ties
 * to the lower index.  mask_dev: DEVICE uint64[d], 8-byte aligned.  Same
 * argument checks and quorum (n >= 2f+1) as gar_aggregate with
 * GAR_TRIMMED_MEAN.  O(n^2) per coordinate: for checking, not the hot path. */
gar_status gar_trimmed_membership(const float* const* grads, int n, int f, int64_t d,
                                  uint64_t* mask_dev, gar_stream_t stream);

/* ---- bf16 gradient rows (R16) ---------------------
 * Not in the paper: its gradients are fp32 tensors.
 * Reading R16: a bf16 input is widened EXACTLY to fp32 and every rule is the
 * fp32 definition applied to the widened values (same canonical order,
 * fp64 averages rounded once to fp32, squared distances, ties to the lower
 * index); outputs stay fp32.  The _dt entry points are the fp32 calls of the
 * same name with a dtype argument and untyped row pointers:
 *   dtype  GAR_F32 (rows are fp32[d]) or GAR_BF16 (rows are bf16[d], the
 *          upper 16 bits of an IEEE fp32, e.g. torch.bfloat16);
 *          anything else -> GAR_ERR_INVALID_ARGUMENT;
 *   grads  host array of n DEVICE pointers, each 16-byte aligned (bf16 rows
 *          are read with 16-byte bulk copies: 8 coordinates per granule);
 *   out    DEVICE fp32[d], 16-byte aligned, not overlapping any row's
 *          [0, d * elem_size) bytes.
 * Argument checks, statuses, workspace sizes (gar_workspace_bytes) and the
 * execution model are those of the fp32 calls. */
typedef enum { GAR_F32 = 0, GAR_BF16 = 1 } gar_dtype;

gar_status gar_aggregate_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m,
                            int64_t d, float* out, int32_t* indices_dev, void* workspace,
                            size_t workspace_bytes, gar_stream_t stream);

gar_status gar_select_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m,
                         int64_t d, int32_t* indices_dev, int* n_selected_host, void* workspace,
                         size_t workspace_bytes, gar_stream_t stream);

gar_status gar_distances_dt(gar_dtype dtype, const void* const* grads, int n, int64_t d, double* D_dev,
                            void* workspace, size_t workspace_bytes, gar_stream_t stream);

gar_status gar_gram_partial_dt(gar_dtype dtype, const void* const* grads, int n, int64_t d_local,
                               double* gram_dev, void* workspace, size_t workspace_bytes,
                               gar_stream_t stream);

gar_status gar_combine_dt(gar_rule rule, gar_dtype dtype, const void* const* grads, int n, int f, int m,
                          int64_t d_local, const int32_t* indices_dev, float* out, gar_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* GARFIELD_B200_GAR_H_ */
