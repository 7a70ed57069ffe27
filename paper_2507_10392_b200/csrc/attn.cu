// Causal flash attention forward / backward for the microbatch executor.
//
// Layout: the fused QKV projection output is read in place — row t of qkv is
// [q(H*D) | k(H*D) | v(H*D)] with row pitch `ld`; sequence b owns rows
// [b*S, (b+1)*S).  O is [T, H*D]; lse is [n_seq, H, S] (natural log).
//
// Round-1 implementation: register-resident online softmax with
// mma.sync.m16n8k16 (bf16 -> fp32) and ldmatrix from XOR-swizzled smem tiles
// loaded by cp.async double buffering.  Backward is split in two passes so no
// atomics are needed: dK/dV per key block, dQ per query block (deterministic).
// The tcgen05/TMEM version is the next step.
#include "common.cuh"
#include "zb_internal.h"

namespace zb {
namespace attn {

constexpr int BM = 64;    // queries per q-tile in the backward passes (4 warps x 16)
constexpr int BN = 64;    // keys per k-tile
constexpr int NW = 4;
constexpr int NT = NW * 32;
constexpr int FW = 8;     // forward / dQ: 8 warps x 16 = 128 queries per CTA
constexpr int FT = FW * 32;
constexpr int FBM = FW * 16;
constexpr float LOG2E = 1.4426950408889634f;

ZB_DEVICE void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
ZB_DEVICE void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
ZB_DEVICE void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

ZB_DEVICE void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
ZB_DEVICE void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
// D += A(16x16, row) * B(16x8, col), bf16 inputs, fp32 accumulators.
ZB_DEVICE void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Swizzled byte offset of (row, col) in a [rows][D] bf16 tile (16-byte chunks XOR row%8).
template <int D>
ZB_DEVICE uint32_t swz(int row, int col) {
  return row * (D * 2) + ((((col >> 3) ^ (row & 7))) << 4) + ((col & 7) << 1);
}

// Copy a [ROWS][D] tile (row-major source with pitch ld) with THREADS threads.
template <int D, int ROWS = 64, int THREADS = NT>
ZB_DEVICE void load_tile(uint8_t* s, const __nv_bfloat16* g, int ld, int tid) {
  constexpr int CH = D / 8;  // 16-byte chunks per row
#pragma unroll
  for (int i = tid; i < ROWS * CH; i += THREADS) {
    const int r = i / CH, c = i % CH;
    cp_async16(s + swz<D>(r, c * 8), g + (size_t)r * ld + c * 8);
  }
}

// A-operand fragment (16 rows x 16 k) from a swizzled tile at (row0, k0).
template <int D>
ZB_DEVICE void ld_a(const uint8_t* s, int row0, int k0, int lane, uint32_t (&a)[4]) {
  const int r = row0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = k0 + (lane >> 4) * 8;
  ldsm_x4(smem_u32(s) + swz<D>(r, c), a[0], a[1], a[2], a[3]);
}
// B fragments for two n8 tiles (rows n0..n0+15 of a [n][k] tile), k0..k0+15 (non-trans).
template <int D>
ZB_DEVICE void ld_b_nk(const uint8_t* s, int n0, int k0, int lane, uint32_t& b00, uint32_t& b01,
                       uint32_t& b10, uint32_t& b11) {
  const int r = n0 + (lane & 7) + (lane >> 4) * 8;
  const int c = k0 + ((lane >> 3) & 1) * 8;
  ldsm_x4(smem_u32(s) + swz<D>(r, c), b00, b01, b10, b11);
}
// B fragments for two n8 tiles (cols n0..n0+15) of a [k][n] tile, k0..k0+15 (trans).
template <int D>
ZB_DEVICE void ld_b_kn(const uint8_t* s, int k0, int n0, int lane, uint32_t& b00, uint32_t& b01,
                       uint32_t& b10, uint32_t& b11) {
  const int r = k0 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int c = n0 + (lane >> 4) * 8;
  ldsm_x4_t(smem_u32(s) + swz<D>(r, c), b00, b01, b10, b11);
}

// ---------------------------------------------------------------- forward
template <int D>
__global__ void __launch_bounds__(FT) fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                __nv_bfloat16* __restrict__ out,
                                                float* __restrict__ lse, int S, int H, int ld,
                                                float scale) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + FBM * D * 2;         // [2][BN][D]
  uint8_t* sV = sK + 2 * BN * D * 2;      // [2][BN][D]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nqb = S / FBM;
  const int qb = nqb - 1 - blockIdx.x;  // heavy (late) query blocks first
  const int h = blockIdx.y, b = blockIdx.z;
  const int HD = H * D;
  const __nv_bfloat16* base = qkv + (size_t)b * S * ld;
  const __nv_bfloat16* gQ = base + (size_t)qb * FBM * ld + h * D;
  const __nv_bfloat16* gK = base + HD + h * D;
  const __nv_bfloat16* gV = base + 2 * HD + h * D;
  const int last_kb = ((qb + 1) * FBM - 1) / BN;  // last key block touching this query block

  load_tile<D, FBM, FT>(sQ, gQ, ld, tid);
  load_tile<D, BN, FT>(sK, gK, ld, tid);
  load_tile<D, BN, FT>(sV, gV, ld, tid);
  cp_commit();

  float o[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const float sl2 = scale * LOG2E;
  uint32_t qf[D / 16][4];
  const int qrow0 = qb * FBM + warp * 16 + (lane >> 2);  // this thread's rows: qrow0, qrow0+8

  for (int kb = 0; kb <= last_kb; ++kb) {
    cp_wait_all();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) ld_a<D>(sQ, warp * 16, kk * 16, lane, qf[kk]);
    }
    if (kb + 1 <= last_kb) {
      const int nb = (kb + 1) & 1;
      load_tile<D, BN, FT>(sK + nb * BN * D * 2, gK + (size_t)(kb + 1) * BN * ld, ld, tid);
      load_tile<D, BN, FT>(sV + nb * BN * D * 2, gV + (size_t)(kb + 1) * BN * ld, ld, tid);
    }
    cp_commit();
    if (kb * BN > qb * FBM + warp * 16 + 15) continue;  // every key of this block is masked for this warp
    const uint8_t* cK = sK + (kb & 1) * BN * D * 2;
    const uint8_t* cV = sV + (kb & 1) * BN * D * 2;
    float s[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < BN / 8; nt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_nk<D>(cK, nt * 8, kk * 16, lane, b00, b01, b10, b11);
        mma16816(s[nt], qf[kk], b00, b01);
        mma16816(s[nt + 1], qf[kk], b10, b11);
      }
    }
    // scale into log2 domain, causal mask on the diagonal block
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = s[nt][e] * sl2;
        if ((kb + 1) * BN > qb * FBM) {
          const int key = kb * BN + nt * 8 + 2 * (lane & 3) + (e & 1);
          const int q = qrow0 + (e >> 1) * 8;
          if (key > q) v = -INFINITY;
        }
        s[nt][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float c0 = exp2f(m0 - mx0), c1 = exp2f(m1 - mx1);
    m0 = mx0;
    m1 = mx1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - m0);
      s[nt][1] = exp2f(s[nt][1] - m0);
      s[nt][2] = exp2f(s[nt][2] - m1);
      s[nt][3] = exp2f(s[nt][3] - m1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * c0 + rs0;
    l1 = l1 * c1 + rs1;
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      o[i][0] *= c0;
      o[i][1] *= c0;
      o[i][2] *= c1;
      o[i][3] *= c1;
    }
    // O += P V
#pragma unroll
    for (int kt = 0; kt < BN / 16; ++kt) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * kt][0], s[2 * kt][1]);
      pa[1] = pack_bf16(s[2 * kt][2], s[2 * kt][3]);
      pa[2] = pack_bf16(s[2 * kt + 1][0], s[2 * kt + 1][1]);
      pa[3] = pack_bf16(s[2 * kt + 1][2], s[2 * kt + 1][3]);
#pragma unroll
      for (int dt = 0; dt < D / 8; dt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_kn<D>(cV, kt * 16, dt * 8, lane, b00, b01, b10, b11);
        mma16816(o[dt], pa, b00, b01);
        mma16816(o[dt + 1], pa, b10, b11);
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = 1.f / l0, i1 = 1.f / l1;
  __nv_bfloat16* o0 = out + ((size_t)b * S + qrow0) * HD + h * D;
  __nv_bfloat16* o1 = o0 + (size_t)8 * HD;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int c = dt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(o0 + c) = pack_bf16(o[dt][0] * i0, o[dt][1] * i0);
    *reinterpret_cast<uint32_t*>(o1 + c) = pack_bf16(o[dt][2] * i1, o[dt][3] * i1);
  }
  if ((lane & 3) == 0) {
    float* lp = lse + ((size_t)b * H + h) * S;
    lp[qrow0] = (m0 + log2f(l0)) / LOG2E;
    lp[qrow0 + 8] = (m1 + log2f(l1)) / LOG2E;
  }
}

// ---------------------------------------------------------------- backward prep
// delta[b,h,q] = sum_d dO[q, h*D+d] * O[q, h*D+d]
__global__ void delta_kernel(const __nv_bfloat16* __restrict__ o,
                             const __nv_bfloat16* __restrict__ dout, float* __restrict__ delta,
                             int T, int S, int H, int D) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T * H) return;
  const int t = warp / H, h = warp % H;
  const __nv_bfloat16* a = o + (size_t)t * H * D + h * D;
  const __nv_bfloat16* g = dout + (size_t)t * H * D + h * D;
  float acc = 0.f;
  for (int i = lane * 2; i < D; i += 64) {
    float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + i));
    float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(g + i));
    acc += x.x * y.x + x.y * y.y;
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    const int b = t / S, q = t % S;
    delta[((size_t)b * H + h) * S + q] = acc;
  }
}

// ---------------------------------------------------------------- backward dK, dV
// One block per (key block, head, seq).  Each warp owns 16 keys and walks the
// query blocks qb >= kb, accumulating dK, dV in registers.
template <int D>
__global__ void __launch_bounds__(NT) bwd_dkdv_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ delta,
    __nv_bfloat16* __restrict__ dqkv, int S, int H, int ld, float scale) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sK = sm;                      // [BN][D]
  uint8_t* sV = sK + BN * D * 2;         // [BN][D]
  uint8_t* sQ = sV + BN * D * 2;         // [2][BM][D]
  uint8_t* sO = sQ + 2 * BM * D * 2;     // [2][BM][D]  (dO)
  float* sL = reinterpret_cast<float*>(sO + 2 * BM * D * 2);  // [2][BM]
  float* sDl = sL + 2 * BM;                                   // [2][BM]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kb = blockIdx.x;  // early key blocks see the most query blocks: launch them first
  const int h = blockIdx.y, b = blockIdx.z;
  const int HD = H * D;
  const __nv_bfloat16* base = qkv + (size_t)b * S * ld;
  const __nv_bfloat16* gQ = base + h * D;
  const __nv_bfloat16* gK = base + (size_t)kb * BN * ld + HD + h * D;
  const __nv_bfloat16* gV = base + (size_t)kb * BN * ld + 2 * HD + h * D;
  const __nv_bfloat16* gO = dout + (size_t)b * S * HD + h * D;
  const float* gL = lse + ((size_t)b * H + h) * S;
  const float* gD = delta + ((size_t)b * H + h) * S;
  const float sl2 = scale * LOG2E;

  load_tile<D>(sK, gK, ld, tid);
  load_tile<D>(sV, gV, ld, tid);
  auto load_q = [&](int qb, int buf) {
    load_tile<D>(sQ + buf * BM * D * 2, gQ + (size_t)qb * BM * ld, ld, tid);
    load_tile<D>(sO + buf * BM * D * 2, gO + (size_t)qb * BM * HD, HD, tid);
    if (tid < BM / 4) {
      cp_async16(sL + buf * BM + tid * 4, gL + qb * BM + tid * 4);
    } else if (tid < BM / 2) {
      const int i = tid - BM / 4;
      cp_async16(sDl + buf * BM + i * 4, gD + qb * BM + i * 4);
    }
  };
  load_q(kb, 0);
  cp_commit();

  float dk[D / 8][4], dv[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[i][e] = dv[i][e] = 0.f;
  const int key0 = kb * BN + warp * 16 + (lane >> 2);  // this thread's keys: key0, key0+8

  for (int qb = kb; qb < S / BM; ++qb) {
    const int buf = (qb - kb) & 1;
    cp_wait_all();
    __syncthreads();
    if (qb + 1 < S / BM) load_q(qb + 1, buf ^ 1);
    cp_commit();
    const uint8_t* cQ = sQ + buf * BM * D * 2;
    const uint8_t* cO = sO + buf * BM * D * 2;
    const float* cL = sL + buf * BM;
    const float* cD = sDl + buf * BM;
    // S^T = K_w Q^T and dP^T = V_w dO^T  (16 keys x 64 queries)
    float st[BM / 8][4], dp[BM / 8][4];
#pragma unroll
    for (int i = 0; i < BM / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t ka[4], va[4];
      ld_a<D>(sK, warp * 16, kk * 16, lane, ka);
      ld_a<D>(sV, warp * 16, kk * 16, lane, va);
#pragma unroll
      for (int nt = 0; nt < BM / 8; nt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_nk<D>(cQ, nt * 8, kk * 16, lane, b00, b01, b10, b11);
        mma16816(st[nt], ka, b00, b01);
        mma16816(st[nt + 1], ka, b10, b11);
        ld_b_nk<D>(cO, nt * 8, kk * 16, lane, b00, b01, b10, b11);
        mma16816(dp[nt], va, b00, b01);
        mma16816(dp[nt + 1], va, b10, b11);
      }
    }
    // P^T = exp(S*scale - lse[q]); dS^T = P^T * (dP^T - delta[q])
#pragma unroll
    for (int nt = 0; nt < BM / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + 2 * (lane & 3) + (e & 1);
        const int key = key0 + (e >> 1) * 8;
        float p = exp2f(st[nt][e] * sl2 - cL[ql] * LOG2E);
        if (qb == kb && key > qb * BM + ql) p = 0.f;
        st[nt][e] = p;
        dp[nt][e] = p * (dp[nt][e] - cD[ql]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
    for (int kt = 0; kt < BM / 16; ++kt) {
      uint32_t pa[4], sa[4];
      pa[0] = pack_bf16(st[2 * kt][0], st[2 * kt][1]);
      pa[1] = pack_bf16(st[2 * kt][2], st[2 * kt][3]);
      pa[2] = pack_bf16(st[2 * kt + 1][0], st[2 * kt + 1][1]);
      pa[3] = pack_bf16(st[2 * kt + 1][2], st[2 * kt + 1][3]);
      sa[0] = pack_bf16(dp[2 * kt][0], dp[2 * kt][1]);
      sa[1] = pack_bf16(dp[2 * kt][2], dp[2 * kt][3]);
      sa[2] = pack_bf16(dp[2 * kt + 1][0], dp[2 * kt + 1][1]);
      sa[3] = pack_bf16(dp[2 * kt + 1][2], dp[2 * kt + 1][3]);
#pragma unroll
      for (int dt = 0; dt < D / 8; dt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_kn<D>(cO, kt * 16, dt * 8, lane, b00, b01, b10, b11);
        mma16816(dv[dt], pa, b00, b01);
        mma16816(dv[dt + 1], pa, b10, b11);
        ld_b_kn<D>(cQ, kt * 16, dt * 8, lane, b00, b01, b10, b11);
        mma16816(dk[dt], sa, b00, b01);
        mma16816(dk[dt + 1], sa, b10, b11);
      }
    }
  }
  __nv_bfloat16* dK0 = dqkv + ((size_t)b * S + key0) * ld + HD + h * D;
  __nv_bfloat16* dV0 = dK0 + HD;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int c = dt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(dK0 + c) = pack_bf16(dk[dt][0] * scale, dk[dt][1] * scale);
    *reinterpret_cast<uint32_t*>(dK0 + (size_t)8 * ld + c) =
        pack_bf16(dk[dt][2] * scale, dk[dt][3] * scale);
    *reinterpret_cast<uint32_t*>(dV0 + c) = pack_bf16(dv[dt][0], dv[dt][1]);
    *reinterpret_cast<uint32_t*>(dV0 + (size_t)8 * ld + c) = pack_bf16(dv[dt][2], dv[dt][3]);
  }
}

// ---------------------------------------------------------------- backward dQ
// One block per (query block, head, seq); walks key blocks kb <= qb.
template <int D>
__global__ void __launch_bounds__(NT) bwd_dq_kernel(
    const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, const float* __restrict__ delta,
    __nv_bfloat16* __restrict__ dqkv, int S, int H, int ld, float scale) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* sQ = sm;                     // [BM][D]
  uint8_t* sO = sQ + BM * D * 2;        // [BM][D]  dO
  uint8_t* sK = sO + BM * D * 2;        // [2][BN][D]
  uint8_t* sV = sK + 2 * BN * D * 2;    // [2][BN][D]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nqb = S / BM;
  const int qb = nqb - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z;
  const int HD = H * D;
  const __nv_bfloat16* base = qkv + (size_t)b * S * ld;
  const __nv_bfloat16* gQ = base + (size_t)qb * BM * ld + h * D;
  const __nv_bfloat16* gK = base + HD + h * D;
  const __nv_bfloat16* gV = base + 2 * HD + h * D;
  const __nv_bfloat16* gO = dout + ((size_t)b * S + qb * BM) * HD + h * D;
  const float sl2 = scale * LOG2E;
  const int qrow0 = qb * BM + warp * 16 + (lane >> 2);
  const float* gL = lse + ((size_t)b * H + h) * S;
  const float* gD = delta + ((size_t)b * H + h) * S;
  const float L0 = gL[qrow0] * LOG2E, L1 = gL[qrow0 + 8] * LOG2E;
  const float D0 = gD[qrow0], D1 = gD[qrow0 + 8];

  load_tile<D>(sQ, gQ, ld, tid);
  load_tile<D>(sO, gO, HD, tid);
  load_tile<D>(sK, gK, ld, tid);
  load_tile<D>(sV, gV, ld, tid);
  cp_commit();
  float dq[D / 8][4];
#pragma unroll
  for (int i = 0; i < D / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  uint32_t qf[D / 16][4], of[D / 16][4];

  for (int kb = 0; kb <= qb; ++kb) {
    cp_wait_all();
    __syncthreads();
    if (kb == 0) {
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        ld_a<D>(sQ, warp * 16, kk * 16, lane, qf[kk]);
        ld_a<D>(sO, warp * 16, kk * 16, lane, of[kk]);
      }
    }
    if (kb + 1 <= qb) {
      const int nb = (kb + 1) & 1;
      load_tile<D>(sK + nb * BN * D * 2, gK + (size_t)(kb + 1) * BN * ld, ld, tid);
      load_tile<D>(sV + nb * BN * D * 2, gV + (size_t)(kb + 1) * BN * ld, ld, tid);
    }
    cp_commit();
    const uint8_t* cK = sK + (kb & 1) * BN * D * 2;
    const uint8_t* cV = sV + (kb & 1) * BN * D * 2;
    float s[BN / 8][4], dp[BN / 8][4];
#pragma unroll
    for (int i = 0; i < BN / 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[i][e] = dp[i][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
#pragma unroll
      for (int nt = 0; nt < BN / 8; nt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_nk<D>(cK, nt * 8, kk * 16, lane, b00, b01, b10, b11);
        mma16816(s[nt], qf[kk], b00, b01);
        mma16816(s[nt + 1], qf[kk], b10, b11);
        ld_b_nk<D>(cV, nt * 8, kk * 16, lane, b00, b01, b10, b11);
        mma16816(dp[nt], of[kk], b00, b01);
        mma16816(dp[nt + 1], of[kk], b10, b11);
      }
    }
#pragma unroll
    for (int nt = 0; nt < BN / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb * BN + nt * 8 + 2 * (lane & 3) + (e & 1);
        const int q = qrow0 + (e >> 1) * 8;
        float p = exp2f(s[nt][e] * sl2 - ((e >> 1) ? L1 : L0));
        if (key > q) p = 0.f;
        dp[nt][e] = p * (dp[nt][e] - ((e >> 1) ? D1 : D0));
      }
    }
    // dQ += dS K   (k = keys, n = dims)
#pragma unroll
    for (int kt = 0; kt < BN / 16; ++kt) {
      uint32_t sa[4];
      sa[0] = pack_bf16(dp[2 * kt][0], dp[2 * kt][1]);
      sa[1] = pack_bf16(dp[2 * kt][2], dp[2 * kt][3]);
      sa[2] = pack_bf16(dp[2 * kt + 1][0], dp[2 * kt + 1][1]);
      sa[3] = pack_bf16(dp[2 * kt + 1][2], dp[2 * kt + 1][3]);
#pragma unroll
      for (int dt = 0; dt < D / 8; dt += 2) {
        uint32_t b00, b01, b10, b11;
        ld_b_kn<D>(cK, kt * 16, dt * 8, lane, b00, b01, b10, b11);
        mma16816(dq[dt], sa, b00, b01);
        mma16816(dq[dt + 1], sa, b10, b11);
      }
    }
  }
  __nv_bfloat16* dQ0 = dqkv + ((size_t)b * S + qrow0) * ld + h * D;
#pragma unroll
  for (int dt = 0; dt < D / 8; ++dt) {
    const int c = dt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(dQ0 + c) = pack_bf16(dq[dt][0] * scale, dq[dt][1] * scale);
    *reinterpret_cast<uint32_t*>(dQ0 + (size_t)8 * ld + c) =
        pack_bf16(dq[dt][2] * scale, dq[dt][3] * scale);
  }
}

template <typename K>
static int prep(K kern, size_t smem) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn: cudaFuncSetAttribute");
  }
  return 0;
}

template <int D>
static int run_fwd(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int ld,
                   float scale, cudaStream_t s) {
  const size_t smem = (size_t)(FBM + 4 * BN) * D * 2;
  if (int rc = prep(fwd_kernel<D>, smem)) return rc;
  fwd_kernel<D><<<dim3(S / FBM, H, n_seq), FT, smem, s>>>(
      (const __nv_bfloat16*)qkv, (__nv_bfloat16*)out, (float*)lse, S, H, ld, scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn_fwd");
}

template <int D>
static int run_bwd(const void* qkv, const void* out, const void* dout, const void* lse,
                   void* dqkv, void* delta, int n_seq, int S, int H, int ld, float scale,
                   cudaStream_t s) {
  const int T = n_seq * S;
  delta_kernel<<<(T * H * 32 + 255) / 256, 256, 0, s>>>(
      (const __nv_bfloat16*)out, (const __nv_bfloat16*)dout, (float*)delta, T, S, H, D);
  const size_t smem_kv = (size_t)(2 * BN + 4 * BM) * D * 2 + 4 * BM * sizeof(float);
  const size_t smem_q = (size_t)(2 * BM + 4 * BN) * D * 2;
  if (int rc = prep(bwd_dkdv_kernel<D>, smem_kv)) return rc;
  if (int rc = prep(bwd_dq_kernel<D>, smem_q)) return rc;
  bwd_dkdv_kernel<D><<<dim3(S / BN, H, n_seq), NT, smem_kv, s>>>(
      (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, (const float*)lse,
      (const float*)delta, (__nv_bfloat16*)dqkv, S, H, ld, scale);
  bwd_dq_kernel<D><<<dim3(S / BM, H, n_seq), NT, smem_q, s>>>(
      (const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dout, (const float*)lse,
      (const float*)delta, (__nv_bfloat16*)dqkv, S, H, ld, scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn_bwd");
}

}  // namespace attn

int launch_attn_delta(const void* o, const void* dout, void* delta, int T, int S, int H, int D,
                      cudaStream_t s) {
  attn::delta_kernel<<<(T * H * 32 + 255) / 256, 256, 0, s>>>(
      (const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, (float*)delta, T, S, H, D);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn delta");
}
}  // namespace zb

using namespace zb;

extern "C" int zb_attn_fwd(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int D,
                           int ld, float scale, cudaStream_t s) {
  if (S % 128) return set_error(ZB_ERR_INVALID, "attn: seq_len must be a multiple of 128");
  if (ld % 8) return set_error(ZB_ERR_INVALID, "attn: ld must be a multiple of 8");
  if (n_seq <= 0) return 0;
  if (D == 64) return attn::run_fwd<64>(qkv, out, lse, n_seq, S, H, ld, scale, s);
  if (D == 128) return attn::run_fwd<128>(qkv, out, lse, n_seq, S, H, ld, scale, s);
  return set_error(ZB_ERR_UNSUPPORTED, "attn: head_dim %d unsupported (64, 128)", D);
}

// dq_accum is unused by the two-pass backward (kept for ABI stability).
extern "C" int zb_attn_bwd(const void* qkv, const void* out, const void* dout, const void* lse,
                           void* dqkv, void* /*dq_accum*/, void* delta, int n_seq, int S, int H,
                           int D, int ld, float scale, cudaStream_t s) {
  if (S % 128) return set_error(ZB_ERR_INVALID, "attn: seq_len must be a multiple of 128");
  if (n_seq <= 0) return 0;
  if (D == 64) return attn::run_bwd<64>(qkv, out, dout, lse, dqkv, delta, n_seq, S, H, ld, scale, s);
  if (D == 128) return attn::run_bwd<128>(qkv, out, dout, lse, dqkv, delta, n_seq, S, H, ld, scale, s);
  return set_error(ZB_ERR_UNSUPPORTED, "attn: head_dim %d unsupported (64, 128)", D);
}
