// membench2.cu — what limits 1D TMA bulk-copy streaming on B200?
// R rows of `chunk` floats per stage, S stages, one consumer pass per stage.
// Variants: number of issuing warps (rows split across warps), number of
// mbarriers per stage, CTAs per SM.  Standalone; not part of libgar.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Rows { const float* p[64]; };
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// PW producer warps (warps W..W+PW-1), each issues rows r with r % PW == its id;
// NB barriers per stage: row r completes on barrier r % NB.
__global__ void k_bulk(Rows rows, int R, int64_t d, int chunk, int S, int PW, int NB, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int W = 8;
  float* buf = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)S * R * chunk * 4);   // [S][NB]
  uint64_t* empty = full + S * NB;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      for (int b = 0; b < NB; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&full[s * NB + b])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&empty[s])), "r"(W));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t ntiles = d / chunk;
  if (warp >= W) {
    const int pw = warp - W;
    if (lane == 0) {
      int s = 0; uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&empty[s])), "r"(ph ^ 1) : "memory");
        // barrier b expects the rows r % NB == b; it is armed by producer warp (b % PW)
        for (int b = pw; b < NB; b += PW) {
          int cnt = 0;
          for (int r = b; r < R; r += NB) ++cnt;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&full[s * NB + b])), "r"(cnt * chunk * 4) : "memory");
        }
        for (int r = pw; r < R; r += PW)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       :: "r"(su32(buf + ((size_t)s * R + r) * chunk)), "l"(rows.p[r] + t * chunk), "r"(chunk * 4), "r"(su32(&full[s * NB + (r % NB)])) : "memory");
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  int s = 0; uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int b = 0; b < NB; ++b)
      asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" :: "r"(su32(&full[s * NB + b])), "r"(ph) : "memory");
    for (int c = threadIdx.x; c < chunk; c += 32 * W) {
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
  const int64_t d = 25557032 / 4096 * 4096;
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* big; CK(cudaMalloc(&big, (size_t)64 * d * 4 + 4096));
  CK(cudaMemset(big, 0, (size_t)64 * d * 4));
  float* out; CK(cudaMalloc(&out, d * 4));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  struct Cfg { int R, chunk, S, PW, NB, occ; };
  Cfg cfgs[] = {
    {31, 256, 3, 1, 1, 1}, {31, 256, 3, 4, 1, 1}, {31, 256, 3, 1, 8, 1}, {31, 256, 3, 4, 4, 1}, {31, 256, 3, 8, 8, 1},
    {31, 128, 6, 1, 1, 1}, {31, 128, 6, 4, 4, 1}, {31, 128, 6, 8, 8, 1},
    {31, 256, 1, 1, 1, 2}, {31, 128, 3, 1, 1, 2}, {31, 128, 3, 4, 4, 2},
    {31, 512, 3, 1, 1, 1}, {31, 512, 3, 4, 4, 1},
    {63, 224, 3, 1, 1, 1}, {63, 224, 3, 4, 4, 1}, {63, 224, 3, 8, 8, 1}, {63, 128, 6, 8, 8, 1},
    {17, 480, 6, 1, 1, 1}, {17, 480, 6, 4, 4, 1},
  };
  for (const Cfg& c : cfgs) {
    Rows rows; for (int i = 0; i < 64; ++i) rows.p[i] = big + (size_t)(i % c.R) * d;
    size_t smem = (size_t)c.S * c.R * c.chunk * 4 + (c.S * c.NB + c.S) * 8;
    if (smem * c.occ > 220 * 1024) { printf("skip R=%d chunk=%d S=%d occ=%d (smem)\n", c.R, c.chunk, c.S, c.occ); continue; }
    int threads = 32 * (8 + c.PW);
    int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bulk, threads, smem));
    int use = c.occ < occ ? c.occ : occ;
    double bytes = (double)c.R * d * 4 + d * 4;
    auto launch = [&] { k_bulk<<<sms * use, threads, smem>>>(rows, c.R, d, c.chunk, c.S, c.PW, c.NB, out); };
    launch(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int it = 0; it < 5; ++it) launch(); cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("R=%2d chunk=%4d (%5d B) S=%d PW=%d NB=%d occ=%d: %7.0f GB/s\n", c.R, c.chunk, c.chunk * 4, c.S, c.PW, c.NB,
           use, bytes / (ms / 5 * 1e-3) / 1e9);
    fflush(stdout);
  }
  return 0;
}
