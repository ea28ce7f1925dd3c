// Shared-memory LDS.128 cost when lanes of a warp share addresses, and the
// FP pipe rates the K6 inner loop can use (FHFMA, FFMA, FFMA2, f16->f32).
// Question for K6: does a warp LDS.128 whose 32 lanes read only D distinct
// 16-byte records cost fewer than 4 wavefronts (so staged-record reuse
// across lanes of one step would cut the shared-memory crossbar work)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/smem_share_bench tools/smem_share_bench.cu
#include <cstdio>
#include <cuda_fp16.h>

// pattern p: lane -> record index inside a 2048-record buffer
__device__ __forceinline__ int rec_of(int pat, int lane) {
  switch (pat) {
    case 0: return lane;                 // 32 distinct, conflict-free
    case 1: return lane >> 1;            // pairs of adjacent lanes share
    case 2: return lane >> 2;            // quads of adjacent lanes
    case 3: return lane & 7;             // 8 distinct, same in every quarter
    case 4: return lane & 15;            // 16 distinct, halves equal
    case 5: return 0;                    // all lanes one record
    case 6: return (lane & 1) ? 100 + (lane >> 1) : (lane >> 1);  // pair-shared, interleaved
    case 7: return (lane * 8) & 31;      // 8-way bank conflict (4 distinct banksets)
    case 8: return ((lane >> 3) << 3) | ((lane & 7) >> 1);  // pairs inside each quarter
    case 9: return (lane & 3) * 8 + (lane >> 2);  // 32 distinct, lane-scrambled
    default: return lane;
  }
}

__global__ void k_lds(int pat, int iters, unsigned* out) {
  extern __shared__ uint4 buf[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned base = (unsigned)__cvta_generic_to_shared(buf) + 16u * (rec_of(pat, lane) + 256 * (warp & 3));
  unsigned a0 = 0, a1 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint4 v;
      // +512*u*16 keeps the same bank pattern but distinct lines per unroll
      asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(base + (u & 1) * 1024 * 16)
                   : "memory");
      a0 += v.x ^ v.y;
      a1 ^= v.z + v.w;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1;
}

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

__global__ void k_ffma2(float* out, int iters) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) {
    float lo = threadIdx.x * 1e-3f + i, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a[i]) : "f"(lo), "f"(hi));
  }
  unsigned long long x, l;
  float xv = 1.0001f, lv = 0.9999f + threadIdx.x * 1e-6f;
  asm("mov.b64 %0, {%1, %1};" : "=l"(x) : "f"(xv));
  asm("mov.b64 %0, {%1, %1};" : "=l"(l) : "f"(lv));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[i]) : "l"(x), "l"(l));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[i]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// f16x2 -> two f32 (cvt) throughput
__global__ void k_cvt(float* out, int iters) {
  unsigned w = 0x3c003c01u + threadIdx.x;
  float s0 = 0, s1 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      __half2 h = *reinterpret_cast<__half2*>(&w);
      float2 f = __half22float2(h);
      s0 += f.x;
      s1 += f.y;
      w += 0x00010001u;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1;
}

int main() {
  unsigned* d;
  float* f;
  cudaMalloc(&d, 148 * 4 * 1024 * sizeof(unsigned));
  cudaMalloc(&f, 148 * 4 * 1024 * sizeof(float));
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 2048 * 16 * 2);
  const char* names[] = {"distinct32", "pairs(l>>1)", "quads(l>>2)", "8dist(l&7)", "16dist(l&15)",
                         "all-one", "pairs-interleaved", "8way-conflict", "pairs-in-quarter",
                         "distinct-scrambled"};
  for (int threads : {256, 512, 1024}) {
    for (int pat = 0; pat < 10; ++pat) {
      const int blocks = 148 * (2048 / threads), iters = 4096;
      k_lds<<<blocks, threads, 2048 * 16 * 2>>>(pat, 16, d);
      cudaEventRecord(e0);
      k_lds<<<blocks, threads, 2048 * 16 * 2>>>(pat, iters, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warp_lds = (double)blocks * (threads / 32) * iters * 8;
      const double cyc = ms * 1e-3 * clk * 1e3;
      printf("LDS.128 %-20s threads=%4d: %.3f SM-cycles per warp LDS.128 (4.0 = 128 B/clk)\n",
             names[pat], threads, cyc * 148 / warp_lds);
    }
  }
  struct K { const char* n; void (*k)(float*, int); double ops; };
  K ks[] = {{"FHFMA", k_fhfma, 16}, {"FFMA2 (2 fma each)", k_ffma2, 8}, {"cvt f16x2->f32x2", k_cvt, 16}};
  for (auto& k : ks) {
    const int blocks = 148 * 4, threads = 512, iters = 8192;
    k.k<<<blocks, threads>>>(f, 16);
    cudaEventRecord(e0);
    k.k<<<blocks, threads>>>(f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_inst = (double)blocks * threads / 32 * iters * k.ops;
    printf("%-22s %.3f warp-instructions per SM-cycle\n", k.n,
           warp_inst / 148 / (ms * 1e-3 * clk * 1e3));
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
