// ffmabench.cu — FFMA issue rate on B200 vs warps per SM sub-partition, with
// NACC independent accumulators per thread (the CUDA-core Gram's register
// blocks), optionally fed by 8-byte shared loads like gram_ccb (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffmabench tools/ffmabench.cu && /tmp/ffmabench
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 2048;

template <int S, bool LOADS, int T>
__global__ void __launch_bounds__(T, 1) bench(float* out, float seed, long long* clk) {
  __shared__ float2 sm[16][256 + 2];
  for (int i = threadIdx.x; i < 16 * 258; i += blockDim.x) (&sm[0][0])[i] = make_float2(seed * i, seed - i);
  __syncthreads();
  float acc[S * S];
#pragma unroll
  for (int e = 0; e < S * S; ++e) acc[e] = 0.f;
  float2 a[S], b[S];
#pragma unroll
  for (int i = 0; i < S; ++i) a[i] = make_float2(seed * (threadIdx.x + i), seed + i), b[i] = make_float2(seed - i, seed * i);
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
    if (LOADS) {
      const int k = (2 * lane + 64 * (it & 3)) & 255;
#pragma unroll
      for (int i = 0; i < S; ++i) a[i] = *reinterpret_cast<const float2*>(&sm[i][k]), b[i] = *reinterpret_cast<const float2*>(&sm[i + 8 - S + S / 2][k]);
    }
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int j = 0; j < S; ++j) acc[i * S + j] = fmaf(a[i].x, b[j].x, acc[i * S + j]);
#pragma unroll
    for (int i = 0; i < S; ++i)
#pragma unroll
      for (int j = 0; j < S; ++j) acc[i * S + j] = fmaf(a[i].y, b[j].y, acc[i * S + j]);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < S * S; ++e) s += acc[e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int S, bool LOADS, int T>
void run() {
  const int threads = T;
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 148 * 8);
  for (int rep = 0; rep < 2; ++rep) bench<S, LOADS, T><<<148, threads>>>(out, 1.0001f, clk);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int b = 0; b < 148; ++b) mx = c[b] > mx ? c[b] : mx;
  const double ffma = double(threads) * ITERS * 2 * S * S;
  printf("S=%2d loads=%d threads=%4d (warps/SMSP %2d): %6.1f FFMA/clk/SM  err=%s\n", S, LOADS, threads, threads / 128,
         ffma / mx, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  run<8, false, 128>(); run<8, false, 256>(); run<8, false, 512>();
  run<8, true, 128>(); run<8, true, 256>(); run<8, true, 512>();
  run<10, false, 128>(); run<10, false, 256>();
  run<10, true, 128>(); run<10, true, 256>();
  run<6, false, 256>(); run<6, false, 512>(); run<6, true, 512>();
  return 0;
}
