// Microbenchmark: tcgen05.mma kind::tf32 issue throughput vs N, A from smem or TMEM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mmabench tools/mmabench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::i8: D s32 (c_format 2), A/B signed 8-bit (format 1), K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// kind::f16: D f32 (c_format 1), A/B fp16 (format 0), K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool ATMEM, bool I8 = false, bool F16 = false>
__global__ void bench(int iters, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  unsigned char* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i & 255);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 64 * 1024);
    constexpr uint32_t id = I8 ? idesc_i8(128, N) : F16 ? idesc_f16(128, N) : idesc_tf32(128, N);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 16; ++kk) {
        const uint64_t bd = sw128_desc(b0 + (kk & 3) * 32);
        const uint32_t acc = (it | kk) ? 1u : 0u;
        if (ATMEM) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                       ::"r"(tb + 256), "r"(tb + 8 * (kk & 7)), "l"(bd), "r"(id), "r"(acc));
        } else if (F16) {
          const uint64_t ad = sw128_desc(a0 + (kk & 3) * 32 + (kk >> 2) * 16384);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tb + 256), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        } else if (I8) {
          const uint64_t ad = sw128_desc(a0 + (kk & 3) * 32 + (kk >> 2) * 16384);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tb + 256), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        } else {
          const uint64_t ad = sw128_desc(a0 + (kk & 3) * 32 + (kk >> 2) * 16384);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(tb + 256), "l"(ad), "l"(bd), "r"(id), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n}"
                   ::"r"(smem_u32(&bar)), "r"(phase));
      phase ^= 1;
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N, bool AT, bool I8 = false, bool F16 = false>
void run() {
  long long* d; cudaMalloc(&d, 148 * 8);
  const int smem = 100 * 1024;
  cudaFuncSetAttribute(bench<N, AT, I8, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  bench<N, AT, I8, F16><<<148, 128, smem>>>(iters, d);
  bench<N, AT, I8, F16><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = (double)h[0] / (iters * 16);
  const int K = I8 ? 32 : F16 ? 16 : 8;
  double macs = 128.0 * N * K;
  printf("%s M=128 N=%3d K=%d A from %s: %6.1f cycles/MMA, %6.0f MAC/clk/SM (%s)\n",
         I8 ? "i8  " : F16 ? "f16 " : "tf32", N, K, AT ? "TMEM" : "smem", cyc, macs / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, false>(); run<128, false>(); run<256, false>();
  run<64, true>(); run<128, true>(); run<256, true>();
  run<64, false, true>(); run<96, false, true>(); run<128, false, true>(); run<256, false, true>();
  run<64, false, false, true>(); run<128, false, false, true>(); run<192, false, false, true>();
  run<256, false, false, true>();
  return 0;
}
