// Microbenchmark: TMEM read throughput of tcgen05.ld.32x32b.x32 with W warps per CTA
// (one CTA per SM, 148 CTAs).  Prints clocks per warp-load and bytes/clk/SM.
#include "common.cuh"
#include <cstdio>
using namespace zb;
__global__ void __launch_bounds__(512, 1) k(int iters, int pass_wait, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(t + (i & 1) * 128, v);
    tmem_ld_wait_regs(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += __uint_as_float(v[j]);
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(slot, 512);
}
int main() {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 4096);
  for (int W : {1, 2, 4, 8, 16}) {
    const int iters = 2000;
    k<<<148, 32 * W>>>(iters, 1, d, s);
    k<<<148, 32 * W>>>(iters, 1, d, s);
    unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)W * iters * 32 * 32 * 4;
    printf("warps %2d: %.1f clk per warp-load, %.1f B/clk/SM (err %s)\n", W, (double)c / iters,
           bytes / c, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
