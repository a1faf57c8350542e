// pipebench.cu — which pipe runs which min/max instruction on B200, and at
// what rate (tools only).  Each kernel runs 8 independent dependency chains
// per thread of one op kind (or two kinds interleaved) and reports thread-ops
// per clock per SM.  If two kinds interleaved reach ~ the sum of their solo
// rates, they issue to different pipes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipebench tools/pipebench.cu && /tmp/pipebench
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ float fmn(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float fmx_nan(float a, float b) {
  float r;
  asm volatile("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ int imn(int a, int b) {
  int r;
  asm volatile("min.s32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t hmn(uint32_t a, uint32_t b) {
  uint32_t r;
  asm volatile("min.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ int vmax3(int a, int b, int c) {
  int r;
  asm volatile("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r + 0 * c;
}
__device__ __forceinline__ float fmn3(float a, float b, float c) {
  float r;
  asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int KIND>
__global__ void bench(float* out, float seed, long long* clk) {
  float f[8];
  int iv[8];
  uint32_t h[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    f[k] = seed * (threadIdx.x + k);
    iv[k] = threadIdx.x * 7 + k;
    h[k] = 0x3f803f80u + threadIdx.x + k;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (KIND == 0) f[k] = fmn(f[k], f[(k + 1) & 7]);                         // FMNMX
      if (KIND == 1) iv[k] = imn(iv[k], iv[(k + 1) & 7]);                      // IMNMX
      if (KIND == 2) h[k] = hmn(h[k], h[(k + 1) & 7]);                         // HMNMX2.BF16
      if (KIND == 3) { f[k] = fmn(f[k], f[(k + 1) & 7]); iv[k] = imn(iv[k], iv[(k + 1) & 7]); }
      if (KIND == 4) { f[k] = fmn(f[k], f[(k + 1) & 7]); h[k] = hmn(h[k], h[(k + 1) & 7]); }
      if (KIND == 5) f[k] = fmx_nan(f[k], f[(k + 1) & 7]);                      // FMNMX.NAN
      if (KIND == 6) iv[k] = vmax3(iv[k], iv[(k + 1) & 7], iv[(k + 2) & 7]);   // VIMNMX s16x2
      if (KIND == 7) { f[k] = fmn(f[k], f[(k + 1) & 7]); iv[k] = vmax3(iv[k], iv[(k + 1) & 7], 0); }
      if (KIND == 8) f[k] = fmn3(f[k], f[(k + 1) & 7], f[(k + 2) & 7]);        // FMNMX3
      if (KIND == 9) f[k] = __fadd_rn(f[k], f[(k + 1) & 7]);                    // FADD (fma pipe)
      if (KIND == 10) { f[k] = fmn(f[k], f[(k + 1) & 7]); iv[k] = iv[k] * 3 + iv[(k + 1) & 7]; }  // FMNMX + IMAD
      if (KIND == 11) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[k]), "f"(f[(k + 1) & 7])); h[k] ^= r; }  // F2FP
      if (KIND == 12) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[k])); f[(k + 1) & 7] += (float)0 * (float)d; iv[k] ^= __double2loint(d); }  // F2F.F64
      if (KIND == 13) { uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[k]), "f"(f[(k + 1) & 7])); h[k] ^= r; f[k] = fmn(f[k], f[(k + 2) & 7]); }  // F2FP + FMNMX
      if (KIND == 14) { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[k])); iv[k] ^= __double2loint(d); uint32_t r; asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(f[(k + 1) & 7]), "f"(f[(k + 2) & 7])); h[k] ^= r; }  // F2F + F2FP
      if (KIND == 16) { double a = __hiloint2double(iv[k], iv[(k + 1) & 7]); double b = __hiloint2double(iv[(k + 2) & 7], iv[k]); double r; asm volatile("min.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b)); iv[k] = __double2loint(r); }  // DMNMX
      if (KIND == 17) { double a = __hiloint2double(iv[k], iv[(k + 1) & 7]); double b = __hiloint2double(iv[(k + 2) & 7], iv[k]); double r; asm volatile("min.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b)); iv[k] = __double2loint(r); f[k] = fmn(f[k], f[(k + 1) & 7]); }  // DMNMX + FMNMX
      if (KIND == 15) { double d = __int_as_float(iv[k]) * 1.0; asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(d), "d"(d), "d"(d)); iv[k] = __double2loint(d); }  // DFMA (+F2F)
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += f[k] + iv[k] + __uint_as_float(h[k]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  const int blocks = 148, threads = 1024;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&clk, blocks * 8);
  const char* names[] = {"FMNMX", "IMNMX", "HMNMX2.BF16", "FMNMX+IMNMX", "FMNMX+HMNMX2", "FMNMX.NAN",
                         "VIMNMX s16x2", "FMNMX+VIMNMX", "FMNMX3", "FADD", "FMNMX+IMAD", "F2FP.PACK",
                         "F2F.F64.F32", "F2FP+FMNMX", "F2F+F2FP", "DFMA(+F2F)", "DMNMX", "DMNMX+FMNMX"};
  int ops[] = {1, 1, 1, 2, 2, 1, 1, 2, 1, 1, 2, 1, 1, 2, 2, 2, 1, 2};
  for (int kind = 0; kind < 18; ++kind) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (kind) {
        case 0: bench<0><<<blocks, threads>>>(out, 1.f, clk); break;
        case 1: bench<1><<<blocks, threads>>>(out, 1.f, clk); break;
        case 2: bench<2><<<blocks, threads>>>(out, 1.f, clk); break;
        case 3: bench<3><<<blocks, threads>>>(out, 1.f, clk); break;
        case 4: bench<4><<<blocks, threads>>>(out, 1.f, clk); break;
        case 5: bench<5><<<blocks, threads>>>(out, 1.f, clk); break;
        case 6: bench<6><<<blocks, threads>>>(out, 1.f, clk); break;
        case 7: bench<7><<<blocks, threads>>>(out, 1.f, clk); break;
        case 8: bench<8><<<blocks, threads>>>(out, 1.f, clk); break;
        case 9: bench<9><<<blocks, threads>>>(out, 1.f, clk); break;
        case 10: bench<10><<<blocks, threads>>>(out, 1.f, clk); break;
        case 11: bench<11><<<blocks, threads>>>(out, 1.f, clk); break;
        case 12: bench<12><<<blocks, threads>>>(out, 1.f, clk); break;
        case 13: bench<13><<<blocks, threads>>>(out, 1.f, clk); break;
        case 14: bench<14><<<blocks, threads>>>(out, 1.f, clk); break;
        case 15: bench<15><<<blocks, threads>>>(out, 1.f, clk); break;
        case 16: bench<16><<<blocks, threads>>>(out, 1.f, clk); break;
        case 17: bench<17><<<blocks, threads>>>(out, 1.f, clk); break;
      }
    }
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int b = 0; b < blocks; ++b) mx = c[b] > mx ? c[b] : mx;
    const double thread_ops = double(threads) * ITERS * 8 * ops[kind];
    printf("%-14s %7.1f thread-ops/clk/SM\n", names[kind], thread_ops / double(mx));
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
