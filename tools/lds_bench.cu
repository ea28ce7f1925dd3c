// Shared-memory LDS.128 throughput vs occupancy and loads in flight.
#include <cstdio>
template <int U>
__global__ void k_lds(float* out, int iters) {
  extern __shared__ uint4 buf[];
  const int n = 2048;
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_uint4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  unsigned a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  unsigned idx = (threadIdx.x * 1) & (n - 1);
  for (int it = 0; it < iters; ++it) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = buf[(idx + u * 97) & (n - 1)];
#pragma unroll
    for (int u = 0; u < U; ++u) { a0 += v[u].x; a1 ^= v[u].y; a2 += v[u].z; a3 ^= v[u].w; }
    idx = (idx + 32 * U) & (n - 1);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(a0 + a1 + a2 + a3);
}
template <int U>
void run(float* d, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2048;
  k_lds<U><<<blocks, threads, 2048 * 16>>>(d, 8);
  cudaEventRecord(e0);
  k_lds<U><<<blocks, threads, 2048 * 16>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double bytes = (double)blocks * threads * iters * U * 16;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("U=%d blocks=%d threads=%d: %.1f B/clk/SM\n", U, blocks, threads,
         bytes / (ms * 1e-3) / 148 / (clk * 1e3));
}
int main() {
  float* d; cudaMalloc(&d, 148 * 2048 * 16 * 4);
  for (int bps : {2, 4, 8}) {
    run<2>(d, 148 * bps, 256); run<4>(d, 148 * bps, 256); run<8>(d, 148 * bps, 256);
  }
  return 0;
}
