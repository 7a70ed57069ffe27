// HBM-bound elementwise / reduction kernels of the transformer step:
// LayerNorm fwd/bwd, token+position embedding fwd/bwd, fused softmax
// cross-entropy (loss + dlogits in one pass over the logits), bias gradients,
// casts. All vectorised 16-byte accesses, warp-shuffle reductions, fp32 math.
#include "common.cuh"
#include "zb_internal.h"

#include <cstdlib>

namespace zb {

// ------------------------------------------------------------------ LayerNorm
// One warp per row; each lane holds its MAXV 16-byte vectors of the row in
// registers, so x is read from HBM once (mean and variance in two register passes).
template <int MAXV>
__global__ void __launch_bounds__(256) layernorm_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y,
    float* __restrict__ mean_out, float* __restrict__ rstd_out, int rows, int d, float eps) {
  pdl_enter();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)row * d);
  const int nv = d >> 3;
  uint4 q[MAXV], qw[MAXV], qb[MAXV];
  float s = 0.f;
  // weight / bias vectors are loaded with the row, so their latency overlaps the
  // two reductions instead of following them
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const uint4* br = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int v = lane + 32 * j;
    q[j] = v < nv ? xr[v] : make_uint4(0, 0, 0, 0);
    if (v < nv) {
      qw[j] = wr[v];
      qb[j] = br[v];
    }
  }
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const uint32_t* qi = &q[j].x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]);
      s += f.x + f.y;
    }
  }
  const float mean = warp_sum(s) / d;
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    if (lane + 32 * j >= nv) continue;
    const uint32_t* qi = &q[j].x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]);
      const float a0 = f.x - mean, a1 = f.y - mean;
      ss += a0 * a0 + a1 * a1;
    }
  }
  const float rstd = rsqrtf(warp_sum(ss) / d + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + (size_t)row * d);
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int v = lane + 32 * j;
    if (v >= nv) continue;
    const uint32_t *qi = &q[j].x, *wi = &qw[j].x, *bi = &qb[j].x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 xv = unpack_bf16(qi[k]), wv = unpack_bf16(wi[k]), bv = unpack_bf16(bi[k]);
      oi[k] = pack_bf16((xv.x - mean) * rstd * wv.x + bv.x, (xv.y - mean) * rstd * wv.y + bv.y);
    }
    yr[v] = o;
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// dx = dres + rstd * (g - mean(g) - xhat * mean(g * xhat)),  g = dy * w
// dw += sum_rows dy * xhat,  db += sum_rows dy.
// Two launches: (1) dx, one warp per row at full occupancy (no
// cross-row state); (2) dw / db as a column reduction over dy and x, structured
// like bias_grad (32 column vectors x 8 row lanes per CTA, 4 loads in flight).
// 75 MB of traffic at HBM speed instead of 50 MB at the fused kernel's
// latency-bound rate (GPT-2 small: 27 us -> ~14 us).
template <int MAXV>
__global__ void __launch_bounds__(256) layernorm_bwd_dx_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const __nv_bfloat16* __restrict__ w, const float* __restrict__ mean_in,
    const float* __restrict__ rstd_in, __nv_bfloat16* dx, const __nv_bfloat16* dres, int rows,
    int d) {
  pdl_enter();
  const int warps = blockDim.x >> 5;
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nv = d >> 3;
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + (size_t)row * d);
  const uint4* xr = reinterpret_cast<const uint4*>(x + (size_t)row * d);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + (size_t)row * d) : nullptr;
  uint4 qd[MAXV], qx[MAXV], qr[MAXV], qw[MAXV];
  const float mean = mean_in[row], rstd = rstd_in[row];
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {   // every load of the row in flight at once
    const int v = lane + 32 * j;
    const bool ok = v < nv;
    qd[j] = ok ? dyr[v] : make_uint4(0, 0, 0, 0);
    qx[j] = ok ? xr[v] : make_uint4(0, 0, 0, 0);
    qr[j] = (ok && rr) ? rr[v] : make_uint4(0, 0, 0, 0);
    qw[j] = ok ? wr[v] : make_uint4(0, 0, 0, 0);
  }
  float sg = 0.f, sgx = 0.f;
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int v = lane + 32 * j;
    if (v >= nv) continue;
    const uint32_t *di = &qd[j].x, *xi = &qx[j].x, *wi = &qw[j].x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]), wv = unpack_bf16(wi[k]);
      const float h0 = (xv.x - mean) * rstd, h1 = (xv.y - mean) * rstd;
      const float g0 = dv.x * wv.x, g1 = dv.y * wv.y;
      sg += g0 + g1;
      sgx += g0 * h0 + g1 * h1;
    }
  }
  const float mg = warp_sum(sg) / d, mgx = warp_sum(sgx) / d;
  uint4* dxr = reinterpret_cast<uint4*>(dx + (size_t)row * d);
#pragma unroll
  for (int j = 0; j < MAXV; ++j) {
    const int v = lane + 32 * j;
    if (v >= nv) continue;
    const uint32_t *di = &qd[j].x, *xi = &qx[j].x, *wi = &qw[j].x, *ri = &qr[j].x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]), wv = unpack_bf16(wi[k]);
      float2 rv = unpack_bf16(ri[k]);
      const float h0 = (xv.x - mean) * rstd, h1 = (xv.y - mean) * rstd;
      oi[k] = pack_bf16(rstd * (dv.x * wv.x - mg - h0 * mgx) + rv.x,
                        rstd * (dv.y * wv.y - mg - h1 * mgx) + rv.y);
    }
    dxr[v] = o;
  }
}

// dw[c] += sum_r dy[r,c] * (x[r,c] - mean[r]) * rstd[r];  db[c] += sum_r dy[r,c]
// EXTRA: also db_res[c] += sum_r dres[r,c] and db_out[c] += sum_r dx[r,c] — the bias
// gradients of the linear layers whose output gradients are dres / dx (GPT block:
// fc2 and attention projection), folded into this column pass.
template <bool EXTRA>
__global__ void __launch_bounds__(256) layernorm_bwd_wb_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, float* __restrict__ dw,
    float* __restrict__ db, const __nv_bfloat16* __restrict__ dres,
    const __nv_bfloat16* __restrict__ dxo, float* __restrict__ db_res, float* __restrict__ db_out,
    int rows, int d, int rows_per_block) {
  pdl_enter();
  constexpr int NV = EXTRA ? 32 : 16;  // accumulated values per column vector
  const int cv = blockIdx.x * 32 + (threadIdx.x & 31);  // column vector (8 cols)
  const int rl = threadIdx.x >> 5;                       // 0..7
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.f;
  const bool ok = cv * 8 < d;
  auto add_row = [&](const uint4& qd, const uint4& qx, float mu, float rs, const uint4& qr,
                     const uint4& qo) {
    const uint32_t *di = &qd.x, *xi = &qx.x, *ri = &qr.x, *oi = &qo.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 dv = unpack_bf16(di[k]), xv = unpack_bf16(xi[k]);
      acc[2 * k] += dv.x * ((xv.x - mu) * rs);
      acc[2 * k + 1] += dv.y * ((xv.y - mu) * rs);
      acc[8 + 2 * k] += dv.x;
      acc[8 + 2 * k + 1] += dv.y;
      if (EXTRA) {
        const float2 rv = unpack_bf16(ri[k]), ov = unpack_bf16(oi[k]);
        acc[16 + 2 * k] += rv.x;
        acc[16 + 2 * k + 1] += rv.y;
        acc[24 + 2 * k] += ov.x;
        acc[24 + 2 * k + 1] += ov.y;
      }
    }
  };
  if (ok) {
    int r = r0 + rl;
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (; r + 24 < r1; r += 32) {
      uint4 qd[4], qx[4], qr[4], qo[4];
      float mu[4], rs[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const size_t o = (size_t)(r + 8 * u) * d + cv * 8;
        qd[u] = *reinterpret_cast<const uint4*>(dy + o);
        qx[u] = *reinterpret_cast<const uint4*>(x + o);
        qr[u] = EXTRA ? *reinterpret_cast<const uint4*>(dres + o) : z;
        qo[u] = EXTRA ? *reinterpret_cast<const uint4*>(dxo + o) : z;
        mu[u] = mean_in[r + 8 * u];
        rs[u] = rstd_in[r + 8 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) add_row(qd[u], qx[u], mu[u], rs[u], qr[u], qo[u]);
    }
    for (; r < r1; r += 8) {
      const size_t o = (size_t)r * d + cv * 8;
      add_row(*reinterpret_cast<const uint4*>(dy + o), *reinterpret_cast<const uint4*>(x + o),
              mean_in[r], rstd_in[r],
              EXTRA ? *reinterpret_cast<const uint4*>(dres + o) : z,
              EXTRA ? *reinterpret_cast<const uint4*>(dxo + o) : z);
    }
  }
  __shared__ float red[8][32][NV + 1];
#pragma unroll
  for (int k = 0; k < NV; ++k) red[rl][threadIdx.x & 31][k] = acc[k];
  __syncthreads();
  // 256 threads reduce the 32 x NV values over the 8 row lanes
  for (int idx = threadIdx.x; idx < 32 * NV; idx += blockDim.x) {
    const int c = idx / NV, k = idx % NV;
    const int col_v = blockIdx.x * 32 + c;
    if (col_v * 8 >= d) continue;
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += red[j][c][k];
    float* dst = k < 8 ? dw : (k < 16 ? db : (k < 24 ? db_res : db_out));
    atomicAdd(&dst[col_v * 8 + (k & 7)], t);
  }
}

// ------------------------------------------------------------------ embedding
__global__ void embedding_fwd_kernel(const int* __restrict__ tok,
                                     const __nv_bfloat16* __restrict__ wte,
                                     const __nv_bfloat16* __restrict__ wpe,
                                     __nv_bfloat16* __restrict__ out, int rows, int d, int seq) {
  pdl_enter();
  const int nv = d >> 3;
  const size_t total = (size_t)rows * nv;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / nv), v = (int)(i % nv);
    const uint4 a = reinterpret_cast<const uint4*>(wte + (size_t)tok[row] * d)[v];
    const uint4 p = wpe ? reinterpret_cast<const uint4*>(wpe + (size_t)(row % seq) * d)[v]
                        : make_uint4(0, 0, 0, 0);  // no learned positions (Llama: RoPE)
    const uint32_t *ai = &a.x, *pi = &p.x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 x = unpack_bf16(ai[k]), y = unpack_bf16(pi[k]);
      oi[k] = pack_bf16(x.x + y.x, x.y + y.y);
    }
    reinterpret_cast<uint4*>(out + (size_t)row * d)[v] = o;
  }
}

__global__ void embedding_bwd_kernel(const int* __restrict__ tok,
                                     const __nv_bfloat16* __restrict__ dout,
                                     float* __restrict__ dwte, float* __restrict__ dwpe, int rows,
                                     int d, int seq) {
  pdl_enter();
  const int nv = d >> 3;
  const size_t total = (size_t)rows * nv;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / nv), v = (int)(i % nv);
    const uint4 g = reinterpret_cast<const uint4*>(dout + (size_t)row * d)[v];
    const uint32_t* gi = &g.x;
    float* te = dwte + (size_t)tok[row] * d + v * 8;
    float* pe = dwpe ? dwpe + (size_t)(row % seq) * d + v * 8 : nullptr;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 x = unpack_bf16(gi[k]);
      atomicAdd(te + 2 * k, x.x);
      atomicAdd(te + 2 * k + 1, x.y);
      if (pe) {
        atomicAdd(pe + 2 * k, x.x);
        atomicAdd(pe + 2 * k + 1, x.y);
      }
    }
  }
}

// ------------------------------------------------------------------ cross-entropy
// One CTA per row: online (max, sum-exp) pass, then dlogits = (softmax - onehot)*scale
// written in place (bf16).  loss_sum += (lse - logit[label]).  label < 0: ignored row;
// label >= V traps (out-of-range class index, as torch's cross_entropy rejects it).
// The label's logit is read before the first barrier: dlogits may alias logits, and
// after the block reduction other warps overwrite the row.
constexpr int XENT_THREADS = 512;
__global__ void __launch_bounds__(XENT_THREADS) xent_kernel(const __nv_bfloat16* logits,
                                                          const int* __restrict__ labels,
                                                          float* __restrict__ loss_sum,
                                                          __nv_bfloat16* dlogits, int V, int ld,
                                                          float scale) {
  pdl_enter();
  const int row = blockIdx.x;
  const __nv_bfloat16* lr = logits + (size_t)row * ld;
  __nv_bfloat16* gr = dlogits + (size_t)row * ld;
  const int label = labels[row];
  if (label >= V) __trap();
  const float label_logit = (threadIdx.x == 0 && label >= 0) ? __bfloat162float(lr[label]) : 0.f;
  const int nv = V >> 3;  // V % 8 == 0 enforced on the host
  float m = -INFINITY, s = 0.f;
  for (int v = threadIdx.x; v < nv; v += XENT_THREADS) {
    uint4 q = reinterpret_cast<const uint4*>(lr)[v];
    const uint32_t* qi = &q.x;
    float vals[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]);
      vals[2 * k] = f.x;
      vals[2 * k + 1] = f.y;
    }
    float lm = vals[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) lm = fmaxf(lm, vals[k]);
    const float nm = fmaxf(m, lm);
    float acc = s * __expf(m - nm);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += __expf(vals[k] - nm);
    m = nm;
    s = acc;
  }
  // block-reduce (m, s)
  __shared__ float sm[XENT_THREADS / 32], ssum[XENT_THREADS / 32];
  __shared__ float s_lse;
  {
    const float wm = warp_max(m);
    float ws = (m == -INFINITY) ? 0.f : s * __expf(m - wm);
    ws = warp_sum(ws);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
      sm[w] = wm;
      ssum[w] = ws;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = XENT_THREADS / 32;
      float a = threadIdx.x < nw ? sm[threadIdx.x] : -INFINITY;
      float bm = warp_max(a);
      float bsum = (threadIdx.x < nw && a != -INFINITY) ? ssum[threadIdx.x] * __expf(a - bm) : 0.f;
      bsum = warp_sum(bsum);
      if (threadIdx.x == 0) s_lse = bm + __logf(bsum);
    }
    __syncthreads();
  }
  const float lse = s_lse;
  if (threadIdx.x == 0 && label >= 0)
    atomicAdd(loss_sum, lse - label_logit);
  const float sc = label >= 0 ? scale : 0.f;
  for (int v = threadIdx.x; v < nv; v += XENT_THREADS) {
    uint4 q = reinterpret_cast<const uint4*>(lr)[v];
    const uint32_t* qi = &q.x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = unpack_bf16(qi[k]);
      const int c = v * 8 + 2 * k;
      float p0 = __expf(f.x - lse) - (c == label ? 1.f : 0.f);
      float p1 = __expf(f.y - lse) - (c + 1 == label ? 1.f : 0.f);
      oi[k] = pack_bf16(p0 * sc, p1 * sc);
    }
    reinterpret_cast<uint4*>(gr)[v] = o;
  }
}

// ------------------------------------------------------------------ bias grad
// db[n] += sum_r dy[r, n].  Block: 32 column-vectors (256 columns) x 8 row lanes;
// each thread keeps 4 row loads in flight.
__global__ void bias_grad_kernel(const __nv_bfloat16* __restrict__ dy, float* __restrict__ db,
                                 int rows, int n, int ld, int rows_per_block) {
  pdl_enter();
  const int cv = blockIdx.x * 32 + (threadIdx.x & 31);  // column vector (8 cols)
  const int rl = threadIdx.x >> 5;                       // 0..7
  const int r0 = blockIdx.y * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool ok = cv * 8 < n;
  if (ok) {
    int r = r0 + rl;
    for (; r + 24 < r1; r += 32) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        q[u] = *reinterpret_cast<const uint4*>(dy + (size_t)(r + 8 * u) * ld + cv * 8);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t* qi = &q[u].x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 f = unpack_bf16(qi[k]);
          acc[2 * k] += f.x;
          acc[2 * k + 1] += f.y;
        }
      }
    }
    for (; r < r1; r += 8) {
      uint4 q = *reinterpret_cast<const uint4*>(dy + (size_t)r * ld + cv * 8);
      const uint32_t* qi = &q.x;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        float2 f = unpack_bf16(qi[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
  }
  __shared__ float red[8][32][9];
#pragma unroll
  for (int k = 0; k < 8; ++k) red[rl][threadIdx.x & 31][k] = acc[k];
  __syncthreads();
  if (rl == 0 && ok) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float t = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) t += red[j][threadIdx.x & 31][k];
      atomicAdd(&db[cv * 8 + k], t);
    }
  }
}

// ------------------------------------------------------------------ small ops
__global__ void cast_f32_bf16_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ d,
                                     int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16(s[i]);
}
__global__ void fill_f32_kernel(float* __restrict__ p, float v, int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void add_bf16_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b,
                                __nv_bfloat16* o, int64_t n) {
  pdl_enter();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    o[i] = __float2bfloat16(__bfloat162float(a[i]) + __bfloat162float(b[i]));
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

static int launched(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, what);
}

}  // namespace zb

using namespace zb;

extern "C" int zb_layernorm_fwd(const void* x, const void* w, const void* b, void* y, void* mean,
                                void* rstd, void* /*reserved*/, int rows, int d, float eps,
                                cudaStream_t s) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "layernorm: d must be a multiple of 8");
  if (rows <= 0) return 0;
  const int threads = 256, per = threads / 32;
  const int vpl = (d / 8 + 31) / 32;
  auto go = [&](auto kern) {
    launch_pdl_k(kern, dim3((rows + per - 1) / per), dim3(threads), 0, s, (const __nv_bfloat16*)x,
                 (const __nv_bfloat16*)w, (const __nv_bfloat16*)b, (__nv_bfloat16*)y, (float*)mean,
                 (float*)rstd, rows, d, eps);
  };
  if (vpl <= 1) go(layernorm_fwd_kernel<1>);
  else if (vpl <= 2) go(layernorm_fwd_kernel<2>);
  else if (vpl <= 3) go(layernorm_fwd_kernel<3>);
  else if (vpl <= 4) go(layernorm_fwd_kernel<4>);
  else if (vpl <= 7) go(layernorm_fwd_kernel<7>);
  else if (vpl <= 10) go(layernorm_fwd_kernel<10>);
  else if (vpl <= 20) go(layernorm_fwd_kernel<20>);
  else return set_error(ZB_ERR_UNSUPPORTED, "layernorm_fwd: d > 5120");
  return launched("layernorm_fwd");
}

// phase: 0 = both launches, 1 = the dx kernel only, 2 = the dw / db column pass only
// (split variant; lets the caller run the column pass on another stream).
static int layernorm_bwd_impl(const void* dy, const void* x, const void* w, const void* mean,
                              const void* rstd, void* dx, void* dw, void* db, const void* dres,
                              void* db_res, void* db_out, int rows, int d, cudaStream_t s,
                              int phase = 0) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "layernorm: d must be a multiple of 8");
  if (d > 5120) return set_error(ZB_ERR_UNSUPPORTED, "layernorm_bwd: d > 5120");
  if (phase < 0 || phase > 2) return set_error(ZB_ERR_INVALID, "layernorm_bwd: phase %d", phase);
  if (rows <= 0) return 0;
  const int threads = 256, per = threads / 32;
  const int vpl = (d / 8 + 31) / 32;  // column vectors per lane
  {
    auto go1 = [&](auto kern) {
      launch_pdl_k(kern, dim3((rows + per - 1) / per), dim3(threads), 0, s,
                   (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, (const __nv_bfloat16*)w,
                   (const float*)mean, (const float*)rstd, (__nv_bfloat16*)dx,
                   (const __nv_bfloat16*)dres, rows, d);
    };
    if (phase == 2) {
    } else if (vpl <= 1) go1(layernorm_bwd_dx_kernel<1>);
    else if (vpl <= 2) go1(layernorm_bwd_dx_kernel<2>);
    else if (vpl <= 3) go1(layernorm_bwd_dx_kernel<3>);
    else if (vpl <= 4) go1(layernorm_bwd_dx_kernel<4>);
    else if (vpl <= 7) go1(layernorm_bwd_dx_kernel<7>);
    else if (vpl <= 10) go1(layernorm_bwd_dx_kernel<10>);
    else go1(layernorm_bwd_dx_kernel<20>);
    if (phase == 1) return launched("layernorm_bwd dx");
    const int cblocks = (d / 8 + 31) / 32;
    int rblocks = (2 * num_sms() + cblocks - 1) / cblocks;
    if (rblocks > rows / 64) rblocks = rows / 64 > 0 ? rows / 64 : 1;
    int rpb = (rows + rblocks - 1) / rblocks;
    rpb = ((rpb + 7) / 8) * 8;
    rblocks = (rows + rpb - 1) / rpb;
    if (db_res || db_out) {
      if (!db_res || !db_out || !dres)
        return set_error(ZB_ERR_INVALID, "layernorm_bwd: db_res / db_out need dres and each other");
      launch_pdl_k(layernorm_bwd_wb_kernel<true>, dim3(cblocks, rblocks), dim3(256), 0, s,
                   (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, (const float*)mean,
                   (const float*)rstd, (float*)dw, (float*)db, (const __nv_bfloat16*)dres,
                   (const __nv_bfloat16*)dx, (float*)db_res, (float*)db_out, rows, d, rpb);
    } else {
      launch_pdl_k(layernorm_bwd_wb_kernel<false>, dim3(cblocks, rblocks), dim3(256), 0, s,
                   (const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, (const float*)mean,
                   (const float*)rstd, (float*)dw, (float*)db, nullptr, nullptr, nullptr, nullptr,
                   rows, d, rpb);
    }
    return launched("layernorm_bwd");
  }
}

extern "C" int zb_layernorm_bwd(const void* dy, const void* x, const void* w, const void* mean,
                                const void* rstd, void* dx, void* dw, void* db, const void* dres,
                                int rows, int d, cudaStream_t s) {
  return layernorm_bwd_impl(dy, x, w, mean, rstd, dx, dw, db, dres, nullptr, nullptr, rows, d, s);
}

extern "C" int zb_layernorm_bwd_ex(const void* dy, const void* x, const void* w, const void* mean,
                                   const void* rstd, void* dx, void* dw, void* db,
                                   const void* dres, void* db_res, void* db_out, int rows, int d,
                                   cudaStream_t s) {
  return layernorm_bwd_impl(dy, x, w, mean, rstd, dx, dw, db, dres, db_res, db_out, rows, d, s);
}

extern "C" int zb_layernorm_bwd_phase(const void* dy, const void* x, const void* w,
                                      const void* mean, const void* rstd, void* dx, void* dw,
                                      void* db, const void* dres, void* db_res, void* db_out,
                                      int rows, int d, int phase, cudaStream_t s) {
  return layernorm_bwd_impl(dy, x, w, mean, rstd, dx, dw, db, dres, db_res, db_out, rows, d, s,
                            phase);
}

extern "C" int zb_embedding_fwd(const void* tok, const void* wte, const void* wpe, void* out,
                                int rows, int d, int seq, cudaStream_t s) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "embedding: d must be a multiple of 8");
  if (rows <= 0) return 0;
  int64_t n = (int64_t)rows * (d / 8);
  launch_pdl_k(embedding_fwd_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, (const int*)tok,
               (const __nv_bfloat16*)wte, (const __nv_bfloat16*)wpe, (__nv_bfloat16*)out, rows, d,
               seq);
  return launched("embedding_fwd");
}

extern "C" int zb_embedding_bwd(const void* tok, const void* dout, void* dwte, void* dwpe,
                                int rows, int d, int seq, cudaStream_t s) {
  if (d % 8) return set_error(ZB_ERR_INVALID, "embedding: d must be a multiple of 8");
  if (rows <= 0) return 0;
  int64_t n = (int64_t)rows * (d / 8);
  launch_pdl_k(embedding_bwd_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, (const int*)tok,
               (const __nv_bfloat16*)dout, (float*)dwte, (float*)dwpe, rows, d, seq);
  return launched("embedding_bwd");
}

// Shared-memory-resident variant (V <= 64K): one CTA per row copies the row into shared
// memory with a single bulk TMA copy, so the logits are read from HBM once and no
// online rescaling is needed: pass 1 row max (no exponentials), pass 2 e =
// exp2((x - max) log2e), summed and written back over the row (bf16), pass 3 dlogits =
// e / sum - onehot (scaled) — one exponential per logit instead of 2.125 (e rounded to
// bf16 before the division: within the bf16 rounding of the stored dlogits).  Two CTAs
// per SM at GPT-2's 50304 columns (98 KB each), so one row's passes overlap the other
// row's copy.
constexpr int XS_THREADS = 512;
constexpr int XS_MAX_V = 65536;
__global__ void __launch_bounds__(XS_THREADS) xent_smem_kernel(
    const __nv_bfloat16* logits, const int* __restrict__ labels, float* __restrict__ loss_sum,
    __nv_bfloat16* dlogits, int V, int ld, float scale) {
  pdl_enter();
  constexpr float LOG2E = 1.4426950408889634f;
  extern __shared__ uint4 row_s[];
  __shared__ uint64_t bar;
  __shared__ float red[XS_THREADS / 32];
  __shared__ float bcast;
  const int row = blockIdx.x;
  const __nv_bfloat16* lr = logits + (size_t)row * ld;
  __nv_bfloat16* gr = dlogits + (size_t)row * ld;
  const int nv = V >> 3;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar, (uint32_t)nv * 16);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(row_s)), "l"(lr), "r"((uint32_t)nv * 16), "r"(smem_u32(&bar))
        : "memory");
  }
  const int label = labels[row];
  if (label >= V) __trap();
  const float label_logit = (threadIdx.x == 0 && label >= 0) ? __bfloat162float(lr[label]) : 0.f;
  __syncthreads();  // barrier initialised before anyone waits on it
  mbar_wait(&bar, 0);
  auto block_reduce = [&](float x, bool is_max) {
    x = is_max ? warp_max(x) : warp_sum(x);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      float y = threadIdx.x < XS_THREADS / 32 ? red[threadIdx.x] : (is_max ? -INFINITY : 0.f);
      y = is_max ? warp_max(y) : warp_sum(y);
      if (threadIdx.x == 0) bcast = y;
    }
    __syncthreads();
    return bcast;
  };
  float mx = -INFINITY;
  for (int v = threadIdx.x; v < nv; v += XS_THREADS) {
    const uint4 q = row_s[v];
    const uint32_t* qi = &q.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(qi[e]);
      mx = fmax3(mx, f.x, f.y);
    }
  }
  const float M = block_reduce(mx, true);
  const float2 l2 = make_float2(LOG2E, LOG2E), nm2 = make_float2(-M * LOG2E, -M * LOG2E);
  float2 acc = make_float2(0.f, 0.f);
  // pass 2: e = exp2((x - max) log2e) in (0, 1], summed, and kept in place of the row
  // (bf16) so the last pass needs no second exponential: p = e / sum
  for (int v = threadIdx.x; v < nv; v += XS_THREADS) {
    const uint4 q = row_s[v];
    const uint32_t* qi = &q.x;
    uint4 eo;
    uint32_t* ei = &eo.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 t = ffma2(unpack_bf16(qi[e]), l2, nm2);
      const float e0 = exp2_fast(t.x), e1 = exp2_fast(t.y);
      acc = fadd2(acc, make_float2(e0, e1));
      ei[e] = pack_bf16(e0, e1);
    }
    row_s[v] = eo;
  }
  const float sum = block_reduce(acc.x + acc.y, false);
  const float lse = M + __logf(sum);
  if (threadIdx.x == 0 && label >= 0) atomicAdd(loss_sum, lse - label_logit);
  const float sc = label >= 0 ? scale : 0.f;
  const float2 inv2 = make_float2(sc / sum, sc / sum);
  for (int v = threadIdx.x; v < nv; v += XS_THREADS) {
    const uint4 q = row_s[v];
    const uint32_t* qi = &q.x;
    uint4 o;
    uint32_t* oi = &o.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 p = fmul2(unpack_bf16(qi[e]), inv2);
      const int c = v * 8 + 2 * e;
      if (c == label) p.x -= sc;
      if (c + 1 == label) p.y -= sc;
      oi[e] = pack_bf16(p.x, p.y);
    }
    reinterpret_cast<uint4*>(gr)[v] = o;
  }
}

extern "C" int zb_xent_fwd_bwd(const void* logits, const void* labels, void* loss_sum,
                               void* dlogits, int rows, int V, int ld, float scale,
                               cudaStream_t s) {
  if (V % 8 || ld % 8) return set_error(ZB_ERR_INVALID, "xent: V and ld must be multiples of 8");
  if (rows <= 0) return 0;
  if (V <= XS_MAX_V && ((uintptr_t)logits & 15) == 0) {
    const int smem = V * 2;
    static int configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
      cudaError_t e = cudaFuncSetAttribute(xent_smem_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, XS_MAX_V * 2);
      if (e != cudaSuccess) return set_cuda_error(e, "xent: cudaFuncSetAttribute");
      configured = XS_MAX_V * 2;
    }
    launch_pdl_k(xent_smem_kernel, dim3(rows), dim3(XS_THREADS), (size_t)smem, s,
                 (const __nv_bfloat16*)logits, (const int*)labels, (float*)loss_sum,
                 (__nv_bfloat16*)dlogits, V, ld, scale);
  } else {  // V > 64K: streaming kernel (online max / sum)
    launch_pdl_k(xent_kernel, dim3(rows), dim3(XENT_THREADS), 0, s, (const __nv_bfloat16*)logits,
                 (const int*)labels, (float*)loss_sum, (__nv_bfloat16*)dlogits, V, ld, scale);
  }
  return launched("xent");
}

extern "C" int zb_bias_grad(const void* dy, void* db, int rows, int n, int ld, cudaStream_t s) {
  if (n % 8 || ld % 8) return set_error(ZB_ERR_INVALID, "bias_grad: n, ld must be multiples of 8");
  if (rows <= 0) return 0;
  const int cblocks = (n / 8 + 31) / 32;
  // ~2 CTAs per SM and >= 64 rows per CTA: each warp then streams >= 8 rows with
  // 4 loads in flight, so the per-CTA reduction is amortised (short CTAs were
  // latency-bound at ~1/6 of HBM bandwidth).
  int rblocks = (2 * num_sms() + cblocks - 1) / cblocks;
  if (rblocks > rows / 64) rblocks = rows / 64 > 0 ? rows / 64 : 1;
  int rpb = (rows + rblocks - 1) / rblocks;
  rpb = ((rpb + 7) / 8) * 8;
  rblocks = (rows + rpb - 1) / rpb;
  launch_pdl_k(bias_grad_kernel, dim3(cblocks, rblocks), dim3(256), 0, s,
               (const __nv_bfloat16*)dy, (float*)db, rows, n, ld, rpb);
  return launched("bias_grad");
}

extern "C" int zb_cast_f32_bf16(const void* src, void* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_pdl_k(cast_f32_bf16_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, (const float*)src,
               (__nv_bfloat16*)dst, n);
  return launched("cast_f32_bf16");
}

extern "C" int zb_fill_f32(void* p, float v, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_pdl_k(fill_f32_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, (float*)p, v, n);
  return launched("fill_f32");
}

extern "C" int zb_add_bf16(const void* a, const void* b, void* o, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  launch_pdl_k(add_bf16_kernel, dim3(grid_for(n, 256)), dim3(256), 0, s, (const __nv_bfloat16*)a,
               (const __nv_bfloat16*)b, (__nv_bfloat16*)o, n);
  return launched("add_bf16");
}
