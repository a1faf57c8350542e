// gram_tc.cu — the pairwise-distance contraction on the 5th-gen tensor cores
// (row a5 of DESIGN.md §1): per-CTA partial Gram matrices of the centred rows,
//     G_ij = sum_k (x_ik - c_k)(x_jk - c_k),
// from which select.cu forms D_ij = G_ii + G_jj - 2 G_ij ("norm correction").
//
// Precision: h = x - c is split as h = hi + lo with
// hi = h truncated to tf32 and lo = h - hi (exact); tcgen05.mma kind::tf32
// multiplies A = [H; L] by B = H (M = 128, N = 64, block-diagonal packing of
// two 64-coordinate blocks when n <= 32, see Cfg):
//     D = [H H^T ; L H^T]   ->   G = H H^T + L H^T + (L H^T)^T
// (3 of the 4 split products; the dropped lo*lo is < 2^-20 relative).  TMEM
// fp32 accumulators are drained every FLUSH tiles into fp64 registers.
//
// Warp roles (one persistent CTA per SM):
//   3 warps     TMA producers: one 1D bulk copy per row per raw stage into the
//               raw ring (rows q mod 3 per warp, one mbarrier each);
//   4-8 warps   converters (warp = 16-coordinate slice of the tile, lane = 8 row
//               groups x 4 chunks): LDS.128 from the raw ring, centring, hi/lo
//               split, STS into the SWIZZLE_128B K-major operand layout,
//               fence.proxy.async, arrive (loads straight from global memory
//               were measured 2x slower: profiles/r1_gram_experiments.md §4);
//   4 or 8 warps epilogue: tcgen05.ld of the accumulator lanes -> fp64 sums
//               (8 when NP = 64: each thread owns half of a 64-column row);
//   last warp   TMEM allocator + single-thread tcgen05.mma issuer.
// n <= kGramCckMaxN goes to the CUDA-core kernels instead (gram_cc.cu,
// gram_cck.cu; launch_gram_partials below).
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "coord_select.h"
#include "elem.cuh"
#include "gram.h"
#include "gram_common.cuh"

// GRAM_EXP (tools/gram_exp.sh only; 0 in the product): 1 = no MMAs issued,
// 2 = converters skip the operand stores, 3 = converters skip all smem work,
// 4 = 1 + 2, 5 = converters skip the proxy fence.  Bottleneck attribution
// (profiles/r1_gram_experiments.md, r2_gram_f16.md);
// results are wrong by construction.
#ifndef GRAM_EXP
#define GRAM_EXP 0
#endif
// NP = 64 ring geometry (A/B knobs for tools/gram_exp.sh; defaults = product)
#ifndef GRAM64_OPS
#define GRAM64_OPS 2
#endif
#ifndef GRAM64_RAW_SUB
#define GRAM64_RAW_SUB 4
#endif
#ifndef GRAM64_RAW_STAGES
#define GRAM64_RAW_STAGES 0
#endif
#ifndef GRAM64_PROD
#define GRAM64_PROD 3
#endif
// NP = 32 ring geometry (A/B knobs; defaults = product)
#ifndef GRAM32_OPS
#define GRAM32_OPS 2
#endif
#ifndef GRAM32_RAW_SUB
#define GRAM32_RAW_SUB 3
#endif

namespace gar {

namespace {

using namespace gram;

template <int NP_, bool BF_ = false>
struct Cfg {
  // BF: bf16 rows (R16): the raw ring holds the bf16 values as
  // copied (2 bytes per coordinate) and the converters widen them exactly to
  // fp32 before centring; everything downstream is the fp32 path.
  static constexpr bool BF = BF_;
  static constexpr int ES = BF ? 2 : 4;          // bytes per coordinate in the raw ring
  static constexpr int BULK_ALIGN = 16 / ES;     // coordinates per 16 bytes (bulk-copy granule)
  static constexpr int NP = NP_;                 // padded row count (8, 16, 32 or 64)
  // Block-diagonal packing: a tile's coordinates are split into BLOCKS blocks
  // that share the MMA's K index; A = [H_0..H_{B-1}; L_0..L_{B-1}] and
  // B = [H_0..H_{B-1}], so the diagonal blocks of D = A B^T are the useful
  // H_b H_b^T and L_b H_b^T (off-diagonal blocks pair different coordinates
  // and are ignored).  NP = 32 -> 2 blocks, M = 128, N = 64: half the MMA
  // instructions of M = 64, N = 32 and the full 128-lane datapath.
  static constexpr int BLOCKS = 64 / NP;         // 8 / 4 / 2 / 1
  static constexpr int M = 2 * NP * BLOCKS;      // 128: H rows of all blocks, then L rows
  static constexpr int N = NP * BLOCKS;          // 64: H rows of all blocks
  static constexpr int CONV_WARPS = (NP <= 32) ? 8 : 4;   // converters: 16*CH coordinates each
  static constexpr int CH = (NP == 8) ? 4 : (NP == 16) ? 2 : 1;  // float4 chunks per lane per tile
  static constexpr int KT = 16 * CH * CONV_WARPS;     // coordinates per tile: 512 / 256 / 128 / 64
  static constexpr int KB = KT / BLOCKS;         // coordinates per block (MMA K extent): 64 in every case
  static constexpr int ATOMS = KB / 32;          // 128-byte K atoms per tile
  static constexpr int ATOM_BYTES = M * 128;     // one K atom of A (8-row groups of 1 KB)
  static constexpr int OP_BYTES = ATOMS * ATOM_BYTES;      // one operand stage (A; B aliases its H rows)
  static constexpr int OP_STAGES = (NP == 64) ? GRAM64_OPS : (NP == 32) ? GRAM32_OPS : 2;
  // Raw ring: one TMA bulk copy per row covers RAW_SUB tiles (1.5 KB / 1 KB per
  // row), issued by PROD_WARPS warps (rows r = p mod PROD_WARPS, one barrier
  // each): bulk-copy issue is limited per request and per issuing warp
  // (tools/membench.cu, membench2.cu).
  static constexpr int PROD_WARPS = (NP == 64) ? GRAM64_PROD : 3;     // 5 or 7 for NP = 64 measured slower (tools/gram_exp.sh)
  static constexpr int RAW_SUB = (NP == 8) ? 1 : (NP == 16) ? 2 : (NP == 32) ? GRAM32_RAW_SUB : GRAM64_RAW_SUB;   // 2 / 2 / 1.5 / 1 KB per row
  static constexpr int RAW_KT = RAW_SUB * KT;    // coordinates per raw stage
  // bytes per raw row (+16: conflict-free LDS.128 per 8-lane phase for fp32
  // and for bf16 at CH >= 2, LDS.64 per 16-lane phase for bf16 at CH = 1)
  static constexpr int RAW_PITCH = RAW_KT * ES + 16;
  // The raw ring holds round_up(n, 8) rows per stage (not NP): its stage count
  // is chosen at launch to fill the shared memory left by the operand stages,
  // so fewer rows buy a deeper ring (n = 35: 3 stages instead of 2; n = 19: 4
  // instead of 3).  Up to RAW_STAGES_MAX stages.
  static constexpr int RAW_STAGES_MAX = 8;
  static constexpr int RAW_STAGES_FIXED = GRAM64_RAW_STAGES;   // (A/B knob: 0 = fill the budget)
  // warp roles: converters | producers | epilogue | MMA = 16 warps (128 registers).
  static constexpr int PRODUCER_WARP = CONV_WARPS;
  static constexpr int EPI_WARP0 = CONV_WARPS + PROD_WARPS;
  static constexpr int EPI_WARPS = (NP <= 32) ? 4 : 8;    // 4 sub-partitions (x column halves, NP = 64)
  static constexpr int EPI_COLS = 32;                     // accumulator columns per epilogue thread
  static constexpr int MMA_WARP = EPI_WARP0 + EPI_WARPS;
  static constexpr int THREADS = (MMA_WARP + 1) * 32;
  static constexpr int TMEM_COLS = 2 * N;        // double-buffered accumulator
  static constexpr int FLUSH = 2;                // tiles accumulated in TMEM (fp32) per fp64 drain
  static constexpr int SMEM_BYTES = 227 * 1024;
  static constexpr int BAR_BYTES = (2 * OP_STAGES + (PROD_WARPS + 1) * RAW_STAGES_MAX + 4) * 8 + 16;
  static constexpr int RAW_REGION = SMEM_BYTES - 1024 /*align*/ - OP_STAGES * OP_BYTES - BAR_BYTES;
  static_assert(THREADS == 16 * 32, "16 warps");
  static_assert(RAW_REGION >= 2 * NP * RAW_PITCH, "two raw stages of NP rows");
  // the epilogue parks T/B over the (then idle) operand + raw rings
  static_assert(2 * NP * (NP + 1) * 8 <= OP_STAGES * OP_BYTES + RAW_REGION, "epilogue T/B parking space");
  static_assert(center_pick_bytes(NP) <= OP_STAGES * OP_BYTES, "centre-pick scratch");
  static_assert(M == 128 && KB % 32 == 0, "tile shape");
};

// STAGE: the fused ingress staging variant (stage rows given); a separate
// instantiation so the plain Gram carries none of its code.
template <int NP, bool STAGE, bool BF>
__global__ void __launch_bounds__(Cfg<NP, BF>::THREADS, 1)
    gram_tc_kernel(const __grid_constant__ RowPtrs rows, int n, int64_t d, int64_t num_tiles,
                   double* __restrict__ partials, int l2_hint, const __grid_constant__ RowPtrs stage,
                   int raw_stages, int raw_bytes) {
  using C = Cfg<NP, BF>;
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment (SWIZZLE_128B) by offsetting the shared array itself, so
  // the compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* ops = base;                                        // OP_STAGES x A operand (SW128)
  unsigned char* raw = base + C::OP_STAGES * C::OP_BYTES;           // raw_stages x [round_up(n, 8)][RAW_PITCH]
  uint64_t* bars = reinterpret_cast<uint64_t*>(raw + C::RAW_REGION);
  uint64_t* raw_full = bars;                          // [RAW_STAGES_MAX][PROD_WARPS] TMA bytes landed
  uint64_t* raw_empty = raw_full + C::RAW_STAGES_MAX * C::PROD_WARPS;   // [RAW_STAGES_MAX] converters done
  uint64_t* op_full = raw_empty + C::RAW_STAGES_MAX;  // [OP_STAGES] operand written
  uint64_t* op_free = op_full + C::OP_STAGES;         // [OP_STAGES] MMAs done reading
  uint64_t* acc_full = op_free + C::OP_STAGES;        // [2]
  uint64_t* acc_empty = acc_full + 2;                 // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;
  // contiguous, balanced tile range [t0, t0 + T) of this CTA
  const int64_t t0 = num_tiles * blockIdx.x / G;
  const int64_t T = num_tiles * (blockIdx.x + 1) / G - t0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < raw_stages; ++s) {
      for (int q = 0; q < C::PROD_WARPS; ++q) mbar_init(&raw_full[s * C::PROD_WARPS + q], 1);
      mbar_init(&raw_empty[s], C::CONV_WARPS);
    }
    for (int s = 0; s < C::OP_STAGES; ++s) {
      mbar_init(&op_full[s], C::CONV_WARPS);
      mbar_init(&op_free[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], C::EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == C::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= C::PRODUCER_WARP && warp < C::PRODUCER_WARP + C::PROD_WARPS) {
    // ====================================================== TMA producers
    // One 1D bulk copy per row per raw stage (RAW_KT*4 bytes, 16-byte aligned,
    // clamped to this CTA's range) into the raw ring.  Producer warp q issues
    // rows r = q (mod PROD_WARPS) and arms barrier q of the stage.
    const int q = warp - C::PRODUCER_WARP;
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      const int my_rows = (n > q) ? (n - q + C::PROD_WARPS - 1) / C::PROD_WARPS : 0;
      const int64_t k_end = ((t0 + T) * C::KT < d) ? (t0 + T) * C::KT : d;
      const int64_t R = (T + C::RAW_SUB - 1) / C::RAW_SUB;
      // ring slot rs and its reuse count, advanced incrementally (the stage
      // count is a launch parameter: no runtime division in the loop)
      int rs = 0;
      uint32_t use = 0;
      for (int64_t j = 0; j < R; ++j, (++rs == raw_stages) ? (rs = 0, ++use) : 0) {
        if (use > 0) mbar_wait_sleep(&raw_empty[rs], (use - 1) & 1);
        const int64_t k0 = t0 * C::KT + j * C::RAW_KT;
        const int64_t cnt = (k_end - k0 < C::RAW_KT) ? k_end - k0 : C::RAW_KT;
        const uint32_t bytes = static_cast<uint32_t>(cnt & ~int64_t(C::BULK_ALIGN - 1)) * C::ES;
        uint64_t* bar = &raw_full[rs * C::PROD_WARPS + q];
        mbar_arrive_expect_tx(bar, bytes * static_cast<uint32_t>(my_rows));
        if (bytes) {
          unsigned char* dst = raw + rs * raw_bytes;
          for (int r = q; r < n; r += C::PROD_WARPS) {
            const void* src = reinterpret_cast<const unsigned char*>(rows.p[r]) + k0 * C::ES;
            if (l2_hint) bulk_g2s(dst + r * C::RAW_PITCH, src, bytes, bar, pol);
            else bulk_g2s_plain(dst + r * C::RAW_PITCH, src, bytes, bar);
          }
        }
      }
    }
  } else if (warp < C::CONV_WARPS) {
    // ====================================================== converters
    // warp = 16-coordinate slice of the tile; lane = (chunk cq = lane/8, row
    // group g = lane%8): rows g, g+8, ... of float4 chunk cq.  Raw rows are
    // padded by 16 B so the 8-row LDS.128 phases are conflict-free; the SW128
    // XOR swizzle does the same for the operand stores.
    // ---- centring row r* of this CTA, picked while the
    // producer's first raw stages are already in flight.  Per-coordinate
    // centring is a translation, so each CTA may pick its own row.
    constexpr int NT = C::CONV_WARPS * 32;
    const int rc = center_pick<NT, NP, BF>(rows, n, d, t0 * C::KT, ops);
    // zero the operand stages once: rows >= n are never written afterwards
    for (int q = threadIdx.x; q < C::OP_STAGES * C::OP_BYTES / 16; q += NT)
      reinterpret_cast<float4*>(ops)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    named_bar(3, NT);
    constexpr int RR = NP / 8;                  // rows per lane
    constexpr int CH = C::CH;                   // float4 chunks per lane per tile
    const int g = lane & 7, cq = lane >> 3;
    // per-lane chunks Q (float4 index within the tile) -> block b, chunk qb
    constexpr int QB = C::KB / 4;               // float4 chunks per block
    int Q[CH];
    uint32_t off_hi[RR][CH], off_lo[RR][CH];
#pragma unroll
    for (int h = 0; h < CH; ++h) {
      Q[h] = (4 * warp + cq) * CH + h;
      const int b = Q[h] / QB, qb = Q[h] % QB;
#pragma unroll
      for (int u = 0; u < RR; ++u) {
        const int r = g + 8 * u;
        off_hi[u][h] = (qb >> 3) * C::ATOM_BYTES + sw128_offset(b * NP + r, qb & 7);
        off_lo[u][h] = (qb >> 3) * C::ATOM_BYTES + sw128_offset(C::N + b * NP + r, qb & 7);
      }
    }
    bool valid[RR];
#pragma unroll
    for (int u = 0; u < RR; ++u) valid[u] = g + 8 * u < n;
    constexpr int CB = 4 * C::ES;                // raw bytes of one 4-coordinate chunk
    const unsigned char* raw_me = raw + Q[0] * CB + g * C::RAW_PITCH;   // chunks Q[0], Q[0]+1, ... are adjacent
    const unsigned char* raw_c = raw + Q[0] * CB + rc * C::RAW_PITCH;
    const int64_t R = (T + C::RAW_SUB - 1) / C::RAW_SUB;
    int rs = 0;
    uint32_t rphase = 0;
    for (int64_t j = 0; j < R; ++j, (++rs == raw_stages) ? (rs = 0, rphase ^= 1) : 0) {
#pragma unroll
      for (int q = 0; q < C::PROD_WARPS; ++q) mbar_wait(&raw_full[rs * C::PROD_WARPS + q], rphase);
      // fused ingress staging (gar_gram_exchange with stage rows): the landed
      // raw stage -- rows that may live on other GPUs -- is also written to
      // this GPU's stage buffers by bulk stores, so the combine that follows
      // reads local memory; the transfer overlaps the Gram tile by tile
      if (STAGE && warp == 0 && lane == 0) {
        const int64_t k0 = t0 * C::KT + j * C::RAW_KT;
        const int64_t k_end = ((t0 + T) * C::KT < d) ? (t0 + T) * C::KT : d;
        const int64_t cnt = (k_end - k0 < C::RAW_KT) ? k_end - k0 : C::RAW_KT;
        const int64_t cb = cnt & ~int64_t(C::BULK_ALIGN - 1);
        const uint32_t bytes = static_cast<uint32_t>(cb) * C::ES;
        if (bytes) {
          for (int r = 0; r < n; ++r)
            bulk_s2g(reinterpret_cast<unsigned char*>(const_cast<float*>(stage.p[r])) + k0 * C::ES,
                     raw + rs * raw_bytes + r * C::RAW_PITCH, bytes);
          bulk_commit();
        }
        for (int64_t k = k0 + cb; k < k0 + cnt; ++k) {   // ragged tail: < 16 bytes per row
          for (int r = 0; r < n; ++r) {
            if constexpr (BF)
              reinterpret_cast<unsigned short*>(const_cast<float*>(stage.p[r]))[k] =
                  reinterpret_cast<const unsigned short*>(rows.p[r])[k];
            else
              const_cast<float*>(stage.p[r])[k] = rows.p[r][k];
          }
        }
      }
#pragma unroll
      for (int sub = 0; sub < C::RAW_SUB; ++sub) {
        const int64_t i = j * C::RAW_SUB + sub;
        if (i >= T) break;
        const int s = static_cast<int>(i % C::OP_STAGES);
        const unsigned char* rt = raw_me + rs * raw_bytes + sub * C::KT * C::ES;
        const unsigned char* rtc = raw_c + rs * raw_bytes + sub * C::KT * C::ES;
        // the tile holding coordinate d-1 may end in a (< 4-coordinate) chunk the
        // bulk copy skipped; only that tile pays for 64-bit bounds checks
        const bool last_tile = (t0 + i + 1) * C::KT > d;
        float4 x[RR][CH], c[CH];
        if (GRAM_EXP == 3) {
          if (i >= C::OP_STAGES) mbar_wait(&op_free[s], static_cast<uint32_t>(i / C::OP_STAGES - 1) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&op_full[s]);
          continue;
        }
        if (!last_tile) {
          if constexpr (!BF) {
#pragma unroll
            for (int h = 0; h < CH; ++h) {
#pragma unroll
              for (int u = 0; u < RR; ++u)   // rows >= n read stale ring data, never stored
                x[u][h] = *reinterpret_cast<const float4*>(rt + u * 8 * C::RAW_PITCH + h * 16);
              c[h] = *reinterpret_cast<const float4*>(rtc + h * 16);
            }
          } else if constexpr (CH == 1) {
#pragma unroll
            for (int u = 0; u < RR; ++u) {
              const uint2 w = *reinterpret_cast<const uint2*>(rt + u * 8 * C::RAW_PITCH);
              x[u][0] = widen2(w.x, w.y);
            }
            const uint2 w = *reinterpret_cast<const uint2*>(rtc);
            c[0] = widen2(w.x, w.y);
          } else {
            // two adjacent chunks per LDS.128 (conflict-free per 8-lane phase)
#pragma unroll
            for (int h = 0; h < CH; h += 2) {
#pragma unroll
              for (int u = 0; u < RR; ++u) {
                const uint4 w = *reinterpret_cast<const uint4*>(rt + u * 8 * C::RAW_PITCH + h * CB);
                x[u][h] = widen2(w.x, w.y);
                x[u][h + 1] = widen2(w.z, w.w);
              }
              const uint4 w = *reinterpret_cast<const uint4*>(rtc + h * CB);
              c[h] = widen2(w.x, w.y);
              c[h + 1] = widen2(w.z, w.w);
            }
          }
        } else {
#pragma unroll
          for (int h = 0; h < CH; ++h) {
            const int64_t k0 = (t0 + i) * C::KT + 4 * Q[h];
            // coordinates below d & ~(BULK_ALIGN-1) arrived by bulk copy; the
            // chunk holding any past it is read from global memory
            const bool ragged = k0 + 4 > (d & ~int64_t(C::BULK_ALIGN - 1));
#pragma unroll
            for (int u = 0; u < RR; ++u) {
              const int r = g + 8 * u;
              x[u][h] = make_float4(0.f, 0.f, 0.f, 0.f);
              if (r < n) x[u][h] = ragged ? load_chunk_t<BF>(rows.p[r], k0, d) : lds_chunk<BF>(rt + u * 8 * C::RAW_PITCH + h * CB);
            }
            c[h] = ragged ? load_chunk_t<BF>(rows.p[rc], k0, d) : lds_chunk<BF>(rtc + h * CB);
          }
        }
#pragma unroll
        for (int h = 0; h < CH; ++h)    // centring c_k = fin(x_{r*,k})
          c[h] = make_float4(fin(c[h].x), fin(c[h].y), fin(c[h].z), fin(c[h].w));
        // split every row unconditionally (rows >= n hold garbage and are simply
        // not stored: their operand rows stay zero), so the compiler can
        // interleave the independent rows instead of branching around each
        float4 hiv[RR][CH], lov[RR][CH];
#pragma unroll
        for (int h = 0; h < CH; ++h) {
#pragma unroll
          for (int u = 0; u < RR; ++u) {
            const float4 xv = x[u][h], cv = c[h];
            float4 hv;
            hv.x = __fsub_rn(xv.x, cv.x); hv.y = __fsub_rn(xv.y, cv.y);
            hv.z = __fsub_rn(xv.z, cv.z); hv.w = __fsub_rn(xv.w, cv.w);
            hiv[u][h] = make_float4(tf32_trunc(hv.x), tf32_trunc(hv.y), tf32_trunc(hv.z), tf32_trunc(hv.w));
            lov[u][h] = make_float4(__fsub_rn(hv.x, hiv[u][h].x), __fsub_rn(hv.y, hiv[u][h].y),
                                    __fsub_rn(hv.z, hiv[u][h].z), __fsub_rn(hv.w, hiv[u][h].w));
          }
        }
        if (i >= C::OP_STAGES) mbar_wait(&op_free[s], static_cast<uint32_t>(i / C::OP_STAGES - 1) & 1);
        unsigned char* At = ops + s * C::OP_BYTES;
#pragma unroll
        for (int h = 0; h < CH; ++h) {
#pragma unroll
          for (int u = 0; u < RR; ++u) {
            if (valid[u] && !(GRAM_EXP == 2 || GRAM_EXP == 4)) {
              *reinterpret_cast<float4*>(At + off_hi[u][h]) = hiv[u][h];
              *reinterpret_cast<float4*>(At + off_lo[u][h]) = lov[u][h];
            }
          }
        }
        if (GRAM_EXP != 5) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&op_full[s]);
      }
      if (STAGE && warp == 0 && lane == 0) bulk_wait_read0();   // stage read out before reuse
      __syncwarp();
      if (lane == 0) mbar_arrive(&raw_empty[rs]);
    }
    if (STAGE && warp == 0 && lane == 0) bulk_wait0();
  } else if (warp == C::MMA_WARP) {
    // ====================================================== MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc<C::M, C::N>();
      const uint32_t op0 = smem_u32(ops);
      for (int64_t i = 0; i < T; ++i) {
        const int s = static_cast<int>(i % C::OP_STAGES);
        const int64_t chunk = i / C::FLUSH;                 // accumulation chunk
        const int buf = static_cast<int>(chunk & 1);
        const bool first = (i % C::FLUSH) == 0;
        const bool last = (i % C::FLUSH) == C::FLUSH - 1 || i == T - 1;
        if (first && chunk >= 2) mbar_wait_sleep(&acc_empty[buf], static_cast<uint32_t>((chunk >> 1) - 1) & 1);
        mbar_wait_sleep(&op_full[s], static_cast<uint32_t>(i / C::OP_STAGES) & 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * C::N;
#pragma unroll
        for (int kk = 0; kk < C::KB / 8; ++kk) {
          const uint32_t a = op0 + s * C::OP_BYTES + (kk >> 2) * C::ATOM_BYTES + (kk & 3) * 32;
          const uint64_t desc = sw128_desc(a);
          if (GRAM_EXP != 1 && GRAM_EXP != 4) mma_tf32(d_tmem, desc, desc, idesc, (first && kk == 0) ? 0u : 1u);
        }
        mma_commit(&op_free[s]);
        if (last) mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ====================================================== epilogue (TMEM -> fp64)
    // Warp -> TMEM sub-partition e (D rows m = 32e + lane).  Rows [0, N) are
    // H_b rows, [N, 2N) L_b rows, b = (m mod N) / NP; the useful columns of
    // block b are [b*NP, (b+1)*NP).  NP = 64: two warps per sub-partition,
    // one per 32-column half.
    const int ew = warp - C::EPI_WARP0;
    const int e = warp & 3;
    const int m = 32 * e + lane;
    const int blk = (m % C::N) / NP;
    // useful columns of block blk: [blk*NP, blk*NP + NP); a 32-column load at
    // col0 covers them starting at offset coff
    const int col0 = (C::BLOCKS > 1) ? (blk * NP / 32) * 32 : (ew >> 2) * 32;
    const int coff = (C::BLOCKS > 1) ? (blk * NP) % 32 : 0;
    double acc[C::EPI_COLS];
#pragma unroll
    for (int j = 0; j < C::EPI_COLS; ++j) acc[j] = 0.0;
    const int64_t nchunks = (T + C::FLUSH - 1) / C::FLUSH;
    for (int64_t i = 0; i < nchunks; ++i) {
      const int buf = static_cast<int>(i & 1);
      mbar_wait_sleep(&acc_full[buf], static_cast<uint32_t>(i >> 1) & 1);
      tc_fence_after();
      float v[C::EPI_COLS];
      tmem_ld32(tmem_base + (static_cast<uint32_t>(32 * e) << 16) + buf * C::N + col0, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
#pragma unroll
      for (int j = 0; j < C::EPI_COLS; ++j) acc[j] += static_cast<double>(v[j]);
    }
    // park T = sum_b H_b H_b^T (TB rows 0..NP-1) and B = sum_b L_b H_b^T
    // (rows NP..2NP-1) in shared memory; blocks are added in fixed order b = 0, 1
    constexpr int EPI_THREADS = C::EPI_WARPS * 32;
    double* TB = reinterpret_cast<double*>(ops);          // [2NP][NP+1]; operand + raw rings are idle now
    const int tb_row = (m < C::N ? 0 : NP) + (m % NP);
    const int tb_col = (C::BLOCKS > 1) ? 0 : col0;
    constexpr int USE = (C::BLOCKS > 1) ? NP : C::EPI_COLS;    // useful accumulator columns
    named_bar(2, EPI_THREADS);
#pragma unroll
    for (int b = 0; b < C::BLOCKS; ++b) {       // fixed order: deterministic fp64 sums
      if (blk == b) {
#pragma unroll
        for (int j = 0; j < C::EPI_COLS; ++j) {
          if (j >= coff && j < coff + USE) {
            double& dst = TB[tb_row * (NP + 1) + tb_col + j - coff];
            dst = (b == 0) ? acc[j] : dst + acc[j];
          }
        }
      }
      named_bar(2, EPI_THREADS);
    }
    double* P = partials + static_cast<size_t>(blockIdx.x) * n * n;
    for (int idx = threadIdx.x - C::EPI_WARP0 * 32; idx < n * n; idx += EPI_THREADS) {
      const int i = idx / n, j = idx % n;
      P[idx] = (TB[i * (NP + 1) + j] + TB[(NP + i) * (NP + 1) + j]) + TB[(NP + j) * (NP + 1) + i];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

template <int NP, bool BF>
cudaError_t launch_np(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                      cudaStream_t stream, const RowPtrs& stage) {
  using C = Cfg<NP, BF>;
  const int64_t tiles = (d + C::KT - 1) / C::KT;
  int grid = num_sms < kGramMaxParts ? num_sms : kGramMaxParts;
  if (tiles < grid) grid = static_cast<int>(tiles > 0 ? tiles : 1);
  int occ = 0;
  const bool staged = stage.p[0] != nullptr;
  auto kern = staged ? gram_tc_kernel<NP, true, BF> : gram_tc_kernel<NP, false, BF>;
  cudaError_t e = cached_occupancy(kern, C::THREADS, C::SMEM_BYTES, &occ);
  if (e != cudaSuccess) return e;
  // raw ring: round_up(n, 8) rows per stage, as many stages as fit.  The
  // converters read all NP rows of a stage (rows >= n are never stored), so the
  // region keeps NP - round_up(n, 8) rows of slack after the last stage.
  const int n8 = (n + 7) / 8 * 8;
  const int raw_bytes = n8 * C::RAW_PITCH;
  int raw_stages = (C::RAW_REGION - (NP - n8) * C::RAW_PITCH) / raw_bytes;
  if (raw_stages > C::RAW_STAGES_MAX) raw_stages = C::RAW_STAGES_MAX;
  if (C::RAW_STAGES_FIXED > 0 && raw_stages > C::RAW_STAGES_FIXED) raw_stages = C::RAW_STAGES_FIXED;
  kern<<<grid, C::THREADS, C::SMEM_BYTES, stream>>>(rp, n, d, tiles, partials, l2_evict_first_enabled(), stage,
                                                     raw_stages, raw_bytes);
  *n_parts = grid;
  return cudaGetLastError();
}

template <bool BF>
cudaError_t launch_gram_t(const float* const* rows, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                          cudaStream_t stream, float* const* stage_rows) {
  RowPtrs rp, st;
  for (int i = 0; i < GAR_MAX_N; ++i) {
    rp.p[i] = (i < n) ? rows[i] : nullptr;
    st.p[i] = (stage_rows && i < n) ? stage_rows[i] : nullptr;
  }
  if (n <= 8) return launch_np<8, BF>(rp, n, d, partials, num_sms, n_parts, stream, st);
  if (n <= 16) return launch_np<16, BF>(rp, n, d, partials, num_sms, n_parts, stream, st);
  if (n <= 32) return launch_np<32, BF>(rp, n, d, partials, num_sms, n_parts, stream, st);
  return launch_np<64, BF>(rp, n, d, partials, num_sms, n_parts, stream, st);
}

}  // namespace

// register-blocked CUDA-core Gram (gram_ccb.cuh, gram_ccb_{f32,bf16}.cu)
cudaError_t launch_gram_ccb_f32(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                                cudaStream_t stream);
cudaError_t launch_gram_ccb_bf16(const RowPtrs& rp, int n, int64_t d, double* partials, int num_sms, int* n_parts,
                                 cudaStream_t stream);

// Kernel choice: CUDA-core FFMA Gram (gram_cc.cu n <= kGramCcMaxN, gram_cck.cu
// n <= kGramCckMaxN, gram_ccb.cuh kGramCcbMinN..kGramCcbMaxN), the tensor-core
// kernel elsewhere (and for the fused ingress staging, which only the
// tensor-core kernel implements).  GAR_GRAM_CC=0
// forces the tensor cores, =1 the CUDA cores up to kGramCckLimit (A/B).
static int gram_cc_forced() {
  static const int v = [] {
    const char* e = getenv("GAR_GRAM_CC");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return v;
}

cudaError_t launch_gram_partials(const float* const* rows, int n, int64_t d, double* partials, int num_sms,
                                 int* n_parts, cudaStream_t stream, float* const* stage_rows, int dtype) {
  const int forced = gram_cc_forced();
  if (!stage_rows && forced != 0) {
    if (n <= kGramCcMaxN) return launch_gram_cc(rows, n, d, partials, num_sms, n_parts, stream, dtype);
    if (n >= kGramCcbMinN && n <= kGramCcbMaxN) {
      RowPtrs rp;
      for (int i = 0; i < GAR_MAX_N; ++i) rp.p[i] = (i < n) ? rows[i] : nullptr;
      return dtype == kBF16 ? launch_gram_ccb_bf16(rp, n, d, partials, num_sms, n_parts, stream)
                            : launch_gram_ccb_f32(rp, n, d, partials, num_sms, n_parts, stream);
    }
    if (n <= (forced == 1 ? kGramCckLimit : kGramCckMaxN))
      return launch_gram_cck(rows, n, d, partials, num_sms, n_parts, stream, dtype);
  }
  if (dtype == kBF16) return launch_gram_t<true>(rows, n, d, partials, num_sms, n_parts, stream, stage_rows);
  if (dtype != kF32) return cudaErrorInvalidValue;
  return launch_gram_t<false>(rows, n, d, partials, num_sms, n_parts, stream, stage_rows);
}

}  // namespace gar
