// Fused AdamW over one rank's uneven fp32 shard (master, exp_avg, exp_avg_sq)
// with the reduce-scattered gradient shard as input; writes the updated bf16
// parameter shard in the same pass (that slice of the layer's flat bf16 buffer
// is what the next AllGather-v broadcasts).  Replaces the reference's modelled
// OptimStep task (hetplan simulate.py:536-550; 1e-10 s/param, costs.py:81).
//
// HBM traffic per element: read master/m/v/grad (16 B) + write master/m/v (12 B)
// + bf16 param (2 B) = 30 B.  float4 vectorised, grid-stride, plus an optional
// per-shard sum of squared gradients reduced with warp shuffles (for logging;
// the interleaved per-ministage optimizer cannot clip by a global norm).
// Update rule follows torch.optim.AdamW (decoupled weight decay, bias-corrected).
#include "adam.cuh"
#include "zb_internal.h"

namespace zb {

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ master,
                                                    float* __restrict__ exp_avg,
                                                    float* __restrict__ exp_avg_sq,
                                                    const float* __restrict__ grad,
                                                    __nv_bfloat16* __restrict__ param,
                                                    float* __restrict__ sumsq, int64_t n,
                                                    AdamParams a) {
  pdl_enter();
  resolve_step(a);
  float ss = 0.f;
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 p = reinterpret_cast<float4*>(master)[i];
    float4 m = reinterpret_cast<float4*>(exp_avg)[i];
    float4 v = reinterpret_cast<float4*>(exp_avg_sq)[i];
    float4 g = reinterpret_cast<const float4*>(grad)[i];
    g.x *= a.grad_scale; g.y *= a.grad_scale; g.z *= a.grad_scale; g.w *= a.grad_scale;
    ss += g.x * g.x + g.y * g.y + g.z * g.z + g.w * g.w;
    adam_elem(p.x, m.x, v.x, g.x, a);
    adam_elem(p.y, m.y, v.y, g.y, a);
    adam_elem(p.z, m.z, v.z, g.z, a);
    adam_elem(p.w, m.w, v.w, g.w, a);
    reinterpret_cast<float4*>(master)[i] = p;
    reinterpret_cast<float4*>(exp_avg)[i] = m;
    reinterpret_cast<float4*>(exp_avg_sq)[i] = v;
    uint2 o;
    o.x = pack_bf16(p.x, p.y);
    o.y = pack_bf16(p.z, p.w);
    reinterpret_cast<uint2*>(param)[i] = o;
  }
  for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float p = master[i], m = exp_avg[i], v = exp_avg_sq[i], g = grad[i] * a.grad_scale;
    ss += g * g;
    adam_elem(p, m, v, g, a);
    master[i] = p;
    exp_avg[i] = m;
    exp_avg_sq[i] = v;
    param[i] = __float2bfloat16(p);
  }
  if (sumsq) {
    __shared__ float red[8];
    ss = warp_sum(ss);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      t = warp_sum(t);
      if (threadIdx.x == 0) atomicAdd(sumsq, t);
    }
  }
}

// ---------------------------------------------------------------- row-split embedding update
// The token-embedding gradient is nonzero only in the rows of this step's tokens.  The
// executor marks those rows (mark[row] = step stamp), clears only them before the
// embedding backward, and splits the table's AdamW: rows NOT marked are updated with
// g = 0 early in the step on a side stream (no gradient read: 26 B/param), the marked
// rows after the backward.  Per element the arithmetic is adam_elem(.., g, ..) exactly as
// in the dense kernel (whose g is 0 for those rows), so the result is bit-identical.
__global__ void embed_mark_kernel(const int* __restrict__ tok, int64_t n, int rows,
                                  int* __restrict__ mark, const int* __restrict__ stamp) {
  pdl_enter();
  const int st = *stamp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = tok[i];
    if (t >= 0 && t < rows) mark[t] = st;
  }
}

// grad rows of the tokens <- 0 (one warp per token; repeated tokens write zeros twice)
__global__ void embed_zero_rows_kernel(const int* __restrict__ tok, int64_t n, int rows,
                                       float* __restrict__ grad, int d) {
  pdl_enter();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += warps) {
    const int t = tok[i];
    if (t < 0 || t >= rows) continue;
    float4* g = reinterpret_cast<float4*>(grad + (size_t)t * d);
    for (int c = lane; c < (d >> 2); c += 32) g[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// AdamW over the rows r of a [rows, d] table with (mark[r] == stamp) == marked; one warp
// per row.  marked == 0: g = 0 and no gradient read.
__global__ void __launch_bounds__(256) adamw_rows_kernel(
    float* __restrict__ master, float* __restrict__ exp_avg, float* __restrict__ exp_avg_sq,
    const float* __restrict__ grad, __nv_bfloat16* __restrict__ param, float* __restrict__ sumsq,
    int rows, int d, const int* __restrict__ mark, int marked, AdamParams a) {
  pdl_enter();
  resolve_step(a);
  const int st = *a.step_dev;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  float ss = 0.f;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    if ((mark[r] == st) != (marked != 0)) continue;
    const size_t base = (size_t)r * d;
    for (int c = lane; c < (d >> 2); c += 32) {
      const size_t i = (base >> 2) + c;
      float4 p = reinterpret_cast<float4*>(master)[i];
      float4 m = reinterpret_cast<float4*>(exp_avg)[i];
      float4 v = reinterpret_cast<float4*>(exp_avg_sq)[i];
      float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
      if (marked) {
        g = reinterpret_cast<const float4*>(grad)[i];
        g.x *= a.grad_scale; g.y *= a.grad_scale; g.z *= a.grad_scale; g.w *= a.grad_scale;
        ss += g.x * g.x + g.y * g.y + g.z * g.z + g.w * g.w;
      }
      adam_elem(p.x, m.x, v.x, g.x, a);
      adam_elem(p.y, m.y, v.y, g.y, a);
      adam_elem(p.z, m.z, v.z, g.z, a);
      adam_elem(p.w, m.w, v.w, g.w, a);
      reinterpret_cast<float4*>(master)[i] = p;
      reinterpret_cast<float4*>(exp_avg)[i] = m;
      reinterpret_cast<float4*>(exp_avg_sq)[i] = v;
      uint2 o;
      o.x = pack_bf16(p.x, p.y);
      o.y = pack_bf16(p.z, p.w);
      reinterpret_cast<uint2*>(param)[i] = o;
    }
  }
  if (sumsq && marked) {
    __shared__ float red[8];
    ss = warp_sum(ss);
    if (lane == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
      float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      t = warp_sum(t);
      if (threadIdx.x == 0) atomicAdd(sumsq, t);
    }
  }
}

}  // namespace zb

using namespace zb;

__global__ void step_inc_kernel(int* step) {
  pdl_enter();
  *step += 1;
}

// step <= 0 with step_dev != NULL: the step number is read from device memory.
static int adamw_impl(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                      void* param_bf16, void* sumsq, int64_t n, float lr, float beta1,
                      float beta2, float eps, float weight_decay, float grad_scale, int step,
                      const int* step_dev, cudaStream_t s) {
  if (n <= 0) return 0;
  if (step < 1 && !step_dev) return set_error(ZB_ERR_INVALID, "adamw: step must be >= 1");
  const uintptr_t al = (uintptr_t)master | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq |
                       (uintptr_t)grad;
  if ((al & 15) || ((uintptr_t)param_bf16 & 7))
    return set_error(ZB_ERR_INVALID, "adamw: shard buffers must be 16-byte aligned");
  AdamParams a;
  a.lr = lr; a.beta1 = beta1; a.beta2 = beta2; a.eps = eps; a.wd = weight_decay;
  a.grad_scale = grad_scale;
  a.step_dev = step_dev;
  if (step < 1) step = 1;
  const double bc1 = 1.0 - pow((double)beta1, step), bc2 = 1.0 - pow((double)beta2, step);
  a.step_size = (float)(lr / bc1);
  a.inv_bc2_sqrt = (float)(1.0 / sqrt(bc2));
  a.decay = 1.f - lr * weight_decay;
  int64_t want = (n / 4 + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  int grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
  launch_pdl_k(adamw_kernel, dim3(grid), dim3(256), 0, s, (float*)master, (float*)exp_avg,
               (float*)exp_avg_sq, (const float*)grad, (__nv_bfloat16*)param_bf16, (float*)sumsq, n,
               a);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "adamw");
}

extern "C" int zb_adamw_shard(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                              void* param_bf16, void* sumsq, int64_t n, float lr, float beta1,
                              float beta2, float eps, float weight_decay, float grad_scale,
                              int step, cudaStream_t s) {
  return adamw_impl(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, n, lr, beta1, beta2,
                    eps, weight_decay, grad_scale, step, nullptr, s);
}

extern "C" int zb_adamw_shard_dstep(void* master, void* exp_avg, void* exp_avg_sq,
                                    const void* grad, void* param_bf16, void* sumsq, int64_t n,
                                    float lr, float beta1, float beta2, float eps,
                                    float weight_decay, float grad_scale, const void* step_dev,
                                    cudaStream_t s) {
  if (!step_dev) return set_error(ZB_ERR_INVALID, "adamw: step_dev is NULL");
  return adamw_impl(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, n, lr, beta1, beta2,
                    eps, weight_decay, grad_scale, 0, (const int*)step_dev, s);
}

extern "C" int zb_step_increment(void* step_dev, cudaStream_t s) {
  launch_pdl_k(step_inc_kernel, dim3(1), dim3(1), 0, s, (int*)step_dev);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "step_increment");
}

extern "C" int zb_embed_mark(const void* tokens, int64_t n, int rows, void* mark,
                             const void* stamp_dev, cudaStream_t s) {
  if (n <= 0) return 0;
  if (!tokens || !mark || !stamp_dev) return set_error(ZB_ERR_INVALID, "embed_mark: NULL pointer");
  const int64_t want = (n + 255) / 256, cap = (int64_t)num_sms() * 8;
  launch_pdl_k(embed_mark_kernel, dim3((int)(want < cap ? want : cap)), dim3(256), 0, s,
               (const int*)tokens, n, rows, (int*)mark, (const int*)stamp_dev);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "embed_mark");
}

extern "C" int zb_embed_zero_rows(const void* tokens, int64_t n, int rows, void* grad, int d,
                                  cudaStream_t s) {
  if (n <= 0) return 0;
  if (!tokens || !grad) return set_error(ZB_ERR_INVALID, "embed_zero_rows: NULL pointer");
  if ((d & 3) || ((uintptr_t)grad & 15))
    return set_error(ZB_ERR_INVALID, "embed_zero_rows: d %% 4 and 16-byte alignment required");
  const int64_t want = (n + 7) / 8, cap = (int64_t)num_sms() * 8;
  launch_pdl_k(embed_zero_rows_kernel, dim3((int)(want < cap ? want : cap)), dim3(256), 0, s,
               (const int*)tokens, n, rows, (float*)grad, d);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "embed_zero_rows");
}

extern "C" int zb_adamw_rows_dstep(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                                   void* param_bf16, void* sumsq, int rows, int d,
                                   const void* mark, int marked, float lr, float beta1,
                                   float beta2, float eps, float weight_decay, float grad_scale,
                                   const void* step_dev, cudaStream_t s) {
  if (rows <= 0) return 0;
  if (!step_dev || !mark || (marked && !grad))
    return set_error(ZB_ERR_INVALID, "adamw_rows: NULL step_dev / mark / grad");
  const uintptr_t al = (uintptr_t)master | (uintptr_t)exp_avg | (uintptr_t)exp_avg_sq |
                       (uintptr_t)grad;
  if ((al & 15) || ((uintptr_t)param_bf16 & 7) || (d & 3))
    return set_error(ZB_ERR_INVALID, "adamw_rows: 16-byte aligned rows of d %% 4 == 0 required");
  const AdamParams a = make_adam_params(lr, beta1, beta2, eps, weight_decay, grad_scale, 0,
                                        (const int*)step_dev);
  const int64_t want = (rows + 7) / 8, cap = (int64_t)num_sms() * 8;
  launch_pdl_k(adamw_rows_kernel, dim3((int)(want < cap ? want : cap)), dim3(256), 0, s,
               (float*)master, (float*)exp_avg, (float*)exp_avg_sq, (const float*)grad,
               (__nv_bfloat16*)param_bf16, (float*)sumsq, rows, d, (const int*)mark, marked, a);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "adamw_rows");
}
