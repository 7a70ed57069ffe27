// Llama-family elementwise kernels (BASELINE configs 4 and 5): RMSNorm fwd/bwd,
// rotary position embedding applied in place on the fused QKV rows (and its
// inverse on the gradients), SwiGLU fwd/bwd.  HBM-bound; 16-byte accesses,
// fp32 math, warp-shuffle reductions.
#include "common.cuh"
#include "zb_internal.h"

namespace zb {

// ------------------------------------------------------------------ RMSNorm
// y = x * rstd * w,  rstd = 1/sqrt(mean(x^2) + eps).  One warp per row.
__global__ void rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ w,
                                   __nv_bfloat16* __restrict__ y, float* __restrict__ rstd_out,
                                   int rows, int d, float eps) {
  pdl_enter();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)row * d);
  const int nv = d >> 3;
  float ss = 0.f;
  for (int v = lane; v < nv; v += 32) {
    uint4 q = xr[v];
    const uint32_t* qi = &q.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
  const float rstd = rsqrtf(warp_sum(ss) / d + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + (size_t)row * d);
  for (int v = lane; v < nv; v += 32) {
    uint4 q = xr[v], qw = wr[v], o;
    const uint32_t *qi = &q.x, *wi = &qw.x;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]), g = unpack_bf16(wi[k]);
      oi[k] = pack_bf16(f.x * rstd * g.x, f.y * rstd * g.y);
    }
    yr[v] = o;
  }
  if (lane == 0) rstd_out[row] = rstd;
}

// dx = dres + rstd * (g - xhat * mean(g * xhat)),  g = dy * w,  xhat = x * rstd
// dw += sum_rows dy * xhat  (smem per-block partials, one atomic per column per block)
__global__ void rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                   const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ w,
                                   const float* __restrict__ rstd_in, __nv_bfloat16* dx,
                                   float* __restrict__ dw, const __nv_bfloat16* dres, int rows,
                                   int d) {
  pdl_enter();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nv = d >> 3;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < rows; row += gridDim.x * warps) {
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + (size_t)row * d);
    const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)row * d);
    const float rstd = rstd_in[row];
    float sgx = 0.f;
    for (int v = lane; v < nv; v += 32) {
      uint4 qd = dyr[v], qx = xr[v], qw = wr[v];
      const uint32_t *di = &qd.x, *xi = &qx.x, *wi = &qw.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]), wv = unpack_bf16(wi[k]);
        const float h0 = xv.x * rstd, h1 = xv.y * rstd;
        sgx += dv.x * wv.x * h0 + dv.y * wv.y * h1;
      }
    }
    const float mgx = warp_sum(sgx) / d;
    uint4* dxr = reinterpret_cast<uint4*>(dx + (size_t)row * d);
    const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + (size_t)row * d) : nullptr;
    for (int v = lane; v < nv; v += 32) {
      uint4 qd = dyr[v], qx = xr[v], qw = wr[v];
      uint4 qr = rr ? rr[v] : make_uint4(0, 0, 0, 0);
      const uint32_t *di = &qd.x, *xi = &qx.x, *wi = &qw.x, *ri = &qr.x;
      uint4 o;
      uint32_t* oi = &o.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]), wv = unpack_bf16(wi[k]);
        float2 rv = rr ? unpack_bf16(ri[k]) : make_float2(0.f, 0.f);
        const float o0 = rstd * (dv.x * wv.x - xv.x * rstd * mgx) + rv.x;
        const float o1 = rstd * (dv.y * wv.y - xv.y * rstd * mgx) + rv.y;
        oi[k] = pack_bf16(o0, o1);
      }
      dxr[v] = o;
    }
  }
}

// dw[c] += sum_r dy[r,c] * x[r,c] * rstd[r]: column reduction (32 column vectors x 8
// row lanes per CTA, 4 loads in flight; the per-row kernel above no longer does
// shared-memory atomics per element).
__global__ void __launch_bounds__(256) rmsnorm_bwd_w_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ rstd_in, float* __restrict__ dw, int rows, int d,
    int rows_per_block) {
  pdl_enter();
  const int cv = blockIdx.x * 32 + (threadIdx.x & 31);
  const int rl = threadIdx.x >> 5;
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (cv * 8 < d) {
    int r = r0 + rl;
    for (; r + 24 < r1; r += 32) {
      uint4 qd[4], qx[4];
      float rs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t o = (size_t)(r + 8 * u) * d + cv * 8;
        qd[u] = *reinterpret_cast<const uint4*>(dy + o);
        qx[u] = *reinterpret_cast<const uint4*>(x + o);
        rs[u] = rstd_in[r + 8 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t *di = &qd[u].x, *xi = &qx[u].x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]);
          acc[2 * k] += dv.x * (xv.x * rs[u]);
          acc[2 * k + 1] += dv.y * (xv.y * rs[u]);
        }
      }
    }
    for (; r < r1; r += 8) {
      const size_t o = (size_t)r * d + cv * 8;
      const uint4 qd = *reinterpret_cast<const uint4*>(dy + o);
      const uint4 qx = *reinterpret_cast<const uint4*>(x + o);
      const float rs = rstd_in[r];
      const uint32_t *di = &qd.x, *xi = &qx.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]);
        acc[2 * k] += dv.x * (xv.x * rs);
        acc[2 * k + 1] += dv.y * (xv.y * rs);
      }
    }
  }
  __shared__ float red[8][32][9];
#pragma unroll
  for (int k = 0; k < 8; ++k) red[rl][threadIdx.x & 31][k] = acc[k];
  __syncthreads();
  if (rl == 0 && cv * 8 < d) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) t += red[j][threadIdx.x & 31][k];
      atomicAdd(&dw[cv * 8 + k], t);
    }
  }
}

// ------------------------------------------------------------------ RoPE
// In place on the q and k parts of fused QKV rows (pitch ld): for each head and
// i < D/2:  (a, b) = (x[i], x[i + D/2]) -> (a cos - b sin, a sin + b cos),
// angle = pos * theta^(-2i/D), pos = row % S.  inverse=1 rotates by -angle
// (the gradient of the rotation).
__global__ void __launch_bounds__(256) rope_kernel(__nv_bfloat16* qkv, int rows, int S, int H,
                                                   int D, int ld, float theta, int inverse) {
  pdl_enter();
  // thread = (row, q/k head, 8 consecutive rotation pairs): two 16-byte loads / stores,
  // inverse frequencies from a per-CTA table
  __shared__ float inv_freq[128];
  const int half = D / 2;
  for (int c = threadIdx.x; c < half; c += blockDim.x)
    inv_freq[c] = exp2f(-(2.f * c / D) * log2f(theta));
  __syncthreads();
  const unsigned groups = half / 8, heads2 = 2 * H;
  const unsigned total = (unsigned)rows * heads2 * groups;  // < 2^31, checked on the host
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned t = i / groups, g = i - t * groups;
    const unsigned row = t / heads2, hh = t - row * heads2;  // hh < H: q heads, else k heads
    const float pos = (float)(row % S);
    __nv_bfloat16* p = qkv + (size_t)row * ld + hh * D + g * 8;
    uint4 qa = *reinterpret_cast<const uint4*>(p), qb = *reinterpret_cast<const uint4*>(p + half);
    uint32_t *ai = &qa.x, *bi = &qb.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = unpack_bf16(ai[k]), b = unpack_bf16(bi[k]);
      float s0, c0, s1, c1;
      sincosf(pos * inv_freq[g * 8 + 2 * k], &s0, &c0);
      sincosf(pos * inv_freq[g * 8 + 2 * k + 1], &s1, &c1);
      if (inverse) {
        s0 = -s0;
        s1 = -s1;
      }
      ai[k] = pack_bf16(a.x * c0 - b.x * s0, a.y * c1 - b.y * s1);
      bi[k] = pack_bf16(a.x * s0 + b.x * c0, a.y * s1 + b.y * c1);
    }
    *reinterpret_cast<uint4*>(p) = qa;
    *reinterpret_cast<uint4*>(p + half) = qb;
  }
}

// ------------------------------------------------------------------ SwiGLU
// gu rows = [gate(f) | up(f)];  out = silu(gate) * up.
// (32-bit index math: the host checks rows * f / 8 < 2^31)
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                  __nv_bfloat16* __restrict__ out, int rows, int f) {
  pdl_enter();
  const unsigned nv = f >> 3;
  const unsigned total = (unsigned)rows * nv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned row = i / nv, v = i - row * nv;
    const __nv_bfloat16* r = gu + (size_t)row * 2 * f;
    const uint4 g = reinterpret_cast<const uint4*>(r)[v];
    const uint4 u = reinterpret_cast<const uint4*>(r + f)[v];
    const uint32_t *gi = &g.x, *ui = &u.x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 a = unpack_bf16(gi[k]), b = unpack_bf16(ui[k]);
      const float s0 = __fdividef(a.x, 1.f + __expf(-a.x)), s1 = __fdividef(a.y, 1.f + __expf(-a.y));
      oi[k] = pack_bf16(s0 * b.x, s1 * b.y);
    }
    reinterpret_cast<uint4*>(out + (size_t)row * f)[v] = o;
  }
}

// dgu = [dgate | dup]:  dgate = dout * up * silu'(gate), dup = dout * silu(gate).
// May run in place (dgu == gu).
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* gu, const __nv_bfloat16* __restrict__ dout,
                                  __nv_bfloat16* dgu, int rows, int f) {
  pdl_enter();
  const unsigned nv = f >> 3;
  const unsigned total = (unsigned)rows * nv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned row = i / nv, v = i - row * nv;
    const __nv_bfloat16* r = gu + (size_t)row * 2 * f;
    const uint4 g = reinterpret_cast<const uint4*>(r)[v];
    const uint4 u = reinterpret_cast<const uint4*>(r + f)[v];
    const uint4 d = reinterpret_cast<const uint4*>(dout + (size_t)row * f)[v];
    const uint32_t *gi = &g.x, *ui = &u.x, *di = &d.x;
    uint4 og, ou;
    uint32_t *ogi = &og.x, *oui = &ou.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 a = unpack_bf16(gi[k]), b = unpack_bf16(ui[k]), dd = unpack_bf16(di[k]);
      const float sg0 = __frcp_rn(1.f + __expf(-a.x)), sg1 = __frcp_rn(1.f + __expf(-a.y));
      const float si0 = a.x * sg0, si1 = a.y * sg1;
      const float ds0 = sg0 * (1.f + a.x * (1.f - sg0)), ds1 = sg1 * (1.f + a.y * (1.f - sg1));
      ogi[k] = pack_bf16(dd.x * b.x * ds0, dd.y * b.y * ds1);
      oui[k] = pack_bf16(dd.x * si0, dd.y * si1);
    }
    __nv_bfloat16* w = dgu + (size_t)row * 2 * f;
    reinterpret_cast<uint4*>(w)[v] = og;
    reinterpret_cast<uint4*>(w + f)[v] = ou;
  }
}

static int grid_for2(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = (long long)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

static int launched2(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, what);
}

}  // namespace zb

using namespace zb;

extern "C" int zb_rmsnorm_fwd(const void* x, const void* w, void* y, void* rstd, int rows, int d,
                              float eps, cudaStream_t s) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "rmsnorm: d must be a multiple of 8");
  if (rows <= 0) return 0;
  launch_pdl_k(rmsnorm_fwd_kernel, dim3((rows + 7) / 8), dim3(256), 0, s, (const __nv_bfloat16*)x,
               (const __nv_bfloat16*)w, (__nv_bfloat16*)y, (float*)rstd, rows, d, eps);
  return launched2("rmsnorm_fwd");
}

extern "C" int zb_rmsnorm_bwd(const void* dy, const void* x, const void* w, const void* rstd,
                              void* dx, void* dw, const void* dres, int rows, int d,
                              cudaStream_t s) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "rmsnorm: d must be a multiple of 8");
  if (rows <= 0) return 0;
  // dx: one warp per row at full occupancy; dw: column reduction
  launch_pdl_k(rmsnorm_bwd_kernel, dim3((rows + 7) / 8), dim3(256), 0, s, (const __nv_bfloat16*)dy,
               (const __nv_bfloat16*)x, (const __nv_bfloat16*)w, (const float*)rstd,
               (__nv_bfloat16*)dx, (float*)dw, (const __nv_bfloat16*)dres, rows, d);
  const int cblocks = (d / 8 + 31) / 32;
  int rblocks = (2 * num_sms() + cblocks - 1) / cblocks;
  if (rblocks > rows / 64) rblocks = rows / 64 > 0 ? rows / 64 : 1;
  int rpb = (rows + rblocks - 1) / rblocks;
  rpb = ((rpb + 7) / 8) * 8;
  rblocks = (rows + rpb - 1) / rpb;
  launch_pdl_k(rmsnorm_bwd_w_kernel, dim3(cblocks, rblocks), dim3(256), 0, s,
               (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, (const float*)rstd, (float*)dw,
               rows, d, rpb);
  return launched2("rmsnorm_bwd");
}

extern "C" int zb_rope(void* qkv, int rows, int S, int H, int D, int ld, float theta, int inverse,
                       cudaStream_t s) {
  if (D % 16 || D > 256) return set_error(ZB_ERR_INVALID, "rope: head_dim must be a multiple of 16, <= 256");
  if (ld % 8 || ((uintptr_t)qkv & 15)) return set_error(ZB_ERR_INVALID, "rope: 16-byte aligned rows needed");
  if (rows <= 0) return 0;
  if ((long long)rows * 2 * H * (D / 16) >= (1ll << 31))
    return set_error(ZB_ERR_UNSUPPORTED, "rope: too many elements for one launch");
  long long n = (long long)rows * 2 * H * (D / 16);
  launch_pdl_k(rope_kernel, dim3(grid_for2(n, 256)), dim3(256), 0, s, (__nv_bfloat16*)qkv, rows, S,
               H, D, ld, theta, inverse);
  return launched2("rope");
}

extern "C" int zb_swiglu_fwd(const void* gu, void* out, int rows, int f, cudaStream_t s) {
  if (f % 8) return set_error(ZB_ERR_INVALID, "swiglu: f must be a multiple of 8");
  if (rows <= 0) return 0;
  if ((long long)rows * (f / 8) >= (1ll << 31))
    return set_error(ZB_ERR_UNSUPPORTED, "swiglu: too many elements for one launch");
  launch_pdl_k(swiglu_fwd_kernel, dim3(grid_for2((long long)rows * (f / 8), 256)), dim3(256), 0, s,
               (const __nv_bfloat16*)gu, (__nv_bfloat16*)out, rows, f);
  return launched2("swiglu_fwd");
}

extern "C" int zb_swiglu_bwd(const void* gu, const void* dout, void* dgu, int rows, int f,
                             cudaStream_t s) {
  if (f % 8) return set_error(ZB_ERR_INVALID, "swiglu: f must be a multiple of 8");
  if (rows <= 0) return 0;
  if ((long long)rows * (f / 8) >= (1ll << 31))
    return set_error(ZB_ERR_UNSUPPORTED, "swiglu: too many elements for one launch");
  launch_pdl_k(swiglu_bwd_kernel, dim3(grid_for2((long long)rows * (f / 8), 256)), dim3(256), 0, s,
               (const __nv_bfloat16*)gu, (const __nv_bfloat16*)dout, (__nv_bfloat16*)dgu, rows, f);
  return launched2("swiglu_bwd");
}
