// common.cuh — shared device helpers for libgar (sm_100a).  Product code.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>

#define GAR_MAX_N 64

namespace gar {

// Row-pointer table passed by value as a kernel parameter (n <= 64 -> 512 B).
struct RowPtrs {
  const float* p[GAR_MAX_N];
};

// Extra output destinations (fused output all-gather): every
// result is also stored at p[j][i] for j < n -- the same offset in the other
// GPUs' replicated output buffers, mapped into this GPU's address space
// (symmetric memory), so the stores travel over NVLink inside the producing
// kernel instead of in a separate all-gather.
//
// Or, with mc set, a multicast address (NVLink SHARP / NVLS):
// one multimem.st per result is replicated by the NVSwitch into every GPU's
// buffer, this GPU's included, so each GPU sends its slice over NVLink once
// instead of once per peer; the local and peer stores are skipped.
//
// Or, with sgd set (the fused server step):
// `out` holds the parameters and each result g updates them in place,
// out[i] = fma(-lr, g, out[i]) (one rounding), instead of being stored.
#define GAR_MAX_PEERS 8
struct OutPtrs {
  float* p[GAR_MAX_PEERS];
  int n;
  float* mc;
  int sgd;
  float lr;
};

__device__ __forceinline__ void mc_store(float* addr, float v) {
  asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void mc_store4(float* addr, float4 v) {
  asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// pv: the caller's preloaded out[i] for the fused server step (ignored otherwise).
__device__ __forceinline__ void store_result(float* out, const OutPtrs& extra, int64_t i, float v, float pv) {
  if (extra.sgd) {
    __stcs(out + i, fmaf(-extra.lr, v, pv));
    return;
  }
  if (extra.mc) {
    mc_store(extra.mc + i, v);
    return;
  }
  __stcs(out + i, v);
  for (int j = 0; j < extra.n; ++j) extra.p[j][i] = v;
}

__device__ __forceinline__ void store_result(float* out, const OutPtrs& extra, int64_t i, float v) {
  store_result(out, extra, i, v, extra.sgd ? __ldcs(out + i) : 0.0f);
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Wait for the phase with parity `parity` to complete.  try_wait with a
// suspend-time hint parks the thread in hardware until the phase completes (or
// the hint expires), so waiting warps do not steal issue slots by polling.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(addr),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// Non-blocking probe: has the phase with parity `parity` completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Same wait, for latency-tolerant waiters (kept as a separate name so the
// policy can differ per role).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); }

// 1D bulk async copy global -> shared (TMA engine), completes on an mbarrier.
// dst, src, bytes must be 16-byte aligned / a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Same copy without an L2 cache-policy operand.
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// 1D bulk async copy shared -> global (TMA engine), bulk-group completion.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the committed bulk stores have finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// ... and completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Canonical value for order statistics (R1): NaN -> +inf, -0 -> +0.
// fminf(NaN, +inf) = +inf (min returns the non-NaN operand); x + 0 maps -0 to +0.
__device__ __forceinline__ float canon(float v) { return __fadd_rn(fminf(v, __int_as_float(0x7f800000)), 0.0f); }

// Host helper: query (and cache) the occupancy of `kern` at (threads, smem).
// The dynamic shared-memory limit is a per-FUNCTION attribute shared by every
// launch configuration of that kernel, so it is raised once per (kernel,
// device) to the device's opt-in maximum rather than to one configuration's
// size (a smaller configuration would otherwise lower it under a larger one).
// Both CUDA calls cost microseconds, which dominate small aggregations.
template <class K>
inline cudaError_t cached_occupancy(K kern, int threads, size_t smem, int* occ) {
  struct Entry {
    const void* fn = nullptr;
    int device = -1;
    int threads = 0;       // 0: the "attribute raised" marker entry
    size_t smem = 0;
    int occ = 0;
  };
  static Entry cache[128];
  static int next = 0;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const void* fn = reinterpret_cast<const void*>(kern);
  bool raised = false;
  for (const Entry& c : cache) {
    if (c.fn != fn || c.device != dev) continue;
    if (c.threads == 0) raised = true;
    if (c.threads == threads && c.smem == smem) {
      *occ = c.occ;
      return cudaSuccess;
    }
  }
  if (!raised) {
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, kern);
    if (e != cudaSuccess) return e;
    int optin = 0;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - static_cast<int>(fa.sharedSizeBytes));
    if (e != cudaSuccess) return e;
    Entry& m = cache[next];
    next = (next + 1) % 128;
    m = Entry{fn, dev, 0, 0, 0};
  }
  int o = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
  if (e != cudaSuccess) return e;
  o = o > 0 ? o : 1;
  Entry& c = cache[next];
  next = (next + 1) % 128;
  c = Entry{fn, dev, threads, smem, o};
  *occ = o;
  return cudaSuccess;
}

}  // namespace gar
