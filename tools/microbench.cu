// Pipe-throughput microbenchmarks for the K6 inner loop on sm_100a:
// FHFMA (fma.rn.f32.f16), FFMA, and conflict-free LDS.128.
#include <cstdio>
#include <cuda_fp16.h>

__device__ __forceinline__ float fhfma(unsigned short a, unsigned short b, float c) {
  float d;
  asm volatile("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(a), "h"(b), "f"(c));
  return d;
}

__global__ void k_fhfma(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  unsigned short x = __half_as_ushort(__float2half(1.0001f));
  unsigned short y = __half_as_ushort(__float2half(0.9999f + threadIdx.x * 1e-6f));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fhfma(x, y, a[i]);
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma(float* out, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float x = 1.0001f, y = 0.9999f + threadIdx.x * 1e-6f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(x, y, a[i]);
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_lds(float* out, int iters) {
  __shared__ uint4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  unsigned acc = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint4 v = buf[(idx + u * 32) & 2047];
      acc += v.x ^ v.w;
    }
    idx += 256;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 64 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_fhfma<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 16;
    printf("FHFMA: %.3f ms, %.1f TFMA/s, %.1f FMA/clk/SM @%d MHz\n", ms, fmas / ms / 1e9,
           fmas / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA : %.3f ms, %.1f TFMA/s, %.1f FMA/clk/SM\n", ms, fmas / ms / 1e9,
           fmas / (ms * 1e-3) / 148 / (clk * 1e3));
    cudaEventRecord(e0);
    k_lds<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)blocks * threads * iters * 8 * 16;
    printf("LDS.128: %.3f ms, %.1f TB/s, %.1f B/clk/SM\n", ms, bytes / ms / 1e9,
           bytes / (ms * 1e-3) / 148 / (clk * 1e3));
  }
  return 0;
}
