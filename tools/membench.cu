// membench.cu — microbenchmark: HBM read bandwidth when a kernel streams R rows
// "in lockstep" (the access pattern of every GAR kernel), for several load
// mechanisms and per-row chunk sizes.  Standalone; not part of libgar.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Rows { const float* p[64]; };

// (a) direct LDG.128: each thread owns CPT float4 chunks of a tile, sums R rows.
template <int CPT>
__global__ void __launch_bounds__(256) k_ldg(Rows rows, int R, int64_t d, float* out) {
  const int64_t tile = 256 * 4 * CPT;
  for (int64_t t0 = blockIdx.x * tile; t0 < d; t0 += gridDim.x * tile) {
    float4 acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = make_float4(0, 0, 0, 0);
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        int64_t k = t0 + (int64_t)(c * 256 + threadIdx.x) * 4;
        if (k + 4 <= d) {
          float4 v = __ldcs(reinterpret_cast<const float4*>(rows.p[r] + k));
          acc[c].x += v.x; acc[c].y += v.y; acc[c].z += v.z; acc[c].w += v.w;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      int64_t k = t0 + (int64_t)(c * 256 + threadIdx.x) * 4;
      if (k + 4 <= d) *reinterpret_cast<float4*>(out + k) = acc[c];
    }
  }
}

// (b) 1D TMA bulk copies of `chunk` floats per row into an S-stage ring, 8 consumer warps.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void __launch_bounds__(288) k_bulk(Rows rows, int R, int64_t d, int chunk, int S, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* buf = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * R * chunk * 4);
  uint64_t* empty = full + S;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&empty[s])), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t ntiles = d / chunk;
  if (warp == 8) {
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&empty[s])), "r"(ph ^ 1) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s])), "r"(R * chunk * 4) : "memory");
        for (int r = 0; r < R; ++r)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su32(buf + ((size_t)s * R + r) * chunk)), "l"(rows.p[r] + t * chunk), "r"(chunk * 4), "r"(su32(&full[s])) : "memory");
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  int s = 0; uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&full[s])), "r"(ph) : "memory");
    for (int c = threadIdx.x; c < chunk; c += 256) {
      float a = 0;
      for (int r = 0; r < R; ++r) a += buf[((size_t)s * R + r) * chunk + c];
      out[t * chunk + c] = a;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(&empty[s])) : "memory");
    if (++s == S) { s = 0; ph ^= 1; }
  }
}

int main() {
  const int64_t d = 25557032 / 4096 * 4096;   // ResNet-50-sized rows
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* big; CK(cudaMalloc(&big, (size_t)64 * d * 4 + 4096));
  CK(cudaMemset(big, 0, (size_t)64 * d * 4));
  float* out; CK(cudaMalloc(&out, d * 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int Rs[] = {1, 8, 17, 31, 63};
  for (int R : Rs) {
    Rows rows; for (int i = 0; i < 64; ++i) rows.p[i] = big + (size_t)(i % R) * d;
    double bytes = (double)R * d * 4 + d * 4;
    auto timeit = [&](auto launch) {
      launch(); CK(cudaDeviceSynchronize());
      cudaEventRecord(a); for (int it = 0; it < 5; ++it) launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b); return bytes / (ms / 5 * 1e-3) / 1e9;
    };
    for (int occ : {2, 4, 8}) {
      printf("R=%2d ldg CPT=1 occ=%d: %7.0f GB/s\n", R, occ, timeit([&] { k_ldg<1><<<sms * occ, 256>>>(rows, R, d, out); }));
      printf("R=%2d ldg CPT=4 occ=%d: %7.0f GB/s\n", R, occ, timeit([&] { k_ldg<4><<<sms * occ, 256>>>(rows, R, d, out); }));
    }
    for (int chunk : {256, 512, 1024, 2048}) {
      for (int S : {2, 3, 4, 6}) {
        size_t smem = (size_t)S * R * chunk * 4 + 2 * S * 8;
        if (smem > 200 * 1024) continue;
        CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bulk, 288, smem));
        printf("R=%2d bulk chunk=%4d (%5d B/row) S=%d occ=%d: %7.0f GB/s\n", R, chunk, chunk * 4, S, occ,
               timeit([&] { k_bulk<<<sms * occ, 288, smem>>>(rows, R, d, chunk, S, out); }));
      }
    }
    fflush(stdout);
  }
  // plain copy reference

  {
    double bytes = 2.0 * d * 4 * 8;
    cudaEventRecord(a);
    for (int it = 0; it < 5; ++it) CK(cudaMemcpyAsync(big + (size_t)8 * d, big, d * 4 * 8, cudaMemcpyDeviceToDevice));
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cudaMemcpy D2D 817 MB: %7.0f GB/s (read+write)\n", bytes / (ms / 5 * 1e-3) / 1e9);
  }
  return 0;
}
