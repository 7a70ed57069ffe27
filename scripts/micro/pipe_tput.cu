// Microbenchmark: per-SM throughput of the softmax instruction mix (ex2.approx, bf16x2
// pack, FFMA, FFMA2, FMNMX) with 16 warps per CTA, one CTA per SM.
#include <cstdio>
#include <cstdint>
template <int OP>
__global__ void __launch_bounds__(512, 1) k(int iters, float seed, unsigned long long* out, float* sink) {
  float a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = seed * (threadIdx.x + j); b[j] = seed - j; }
  uint32_t u = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j]));
      if (OP == 1) { uint32_t p; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(a[j]), "f"(b[j])); u ^= p; }
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[j]) : "f"(b[j]));
      if (OP == 3) asm volatile("{.reg .b64 t; mov.b64 t, {%0,%1}; fma.rn.f32x2 t, t, t, t; mov.b64 {%0,%1}, t;}" : "+f"(a[j]), "+f"(b[j]));
      if (OP == 4) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[j]) : "f"(b[j]));
      if (OP == 5) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[j])); uint32_t p; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(a[j]), "f"(b[j])); u ^= p; }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  float s = u;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j] + b[j];
  if (s == 1.2345f) sink[threadIdx.x] = s;
}
template <int OP> void run(const char* name, unsigned long long* d, float* s) {
  const int iters = 4000, W = 16;
  k<OP><<<148, 32 * W>>>(iters, 0.001f, d, s);
  k<OP><<<148, 32 * W>>>(iters, 0.001f, d, s);
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double ops = (double)W * 32 * iters * 8;
  printf("%-12s %.2f thread-ops/clk/SM  (%s)\n", name, ops / c, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d; float* s;
  cudaMalloc(&d, 8); cudaMalloc(&s, 4096);
  run<0>("ex2", d, s); run<1>("cvt bf16x2", d, s); run<2>("ffma", d, s); run<3>("ffma2", d, s);
  run<4>("fmax", d, s); run<5>("ex2+cvt", d, s);
  return 0;
}
