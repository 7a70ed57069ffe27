// Causal flash-attention backward on tcgen05 / TMEM / TMA (sm_100a).
//
// Two kernels, no atomics (deterministic):
//   dq:   one CTA per 128-query tile; per 128-key block j (j <= tile):
//           S = Q K_j^T, dP = dO V_j^T           (tensor core -> TMEM)
//           dS = P * (dP - delta),  P = exp(S*scale - lse)   (one thread per query row)
//           dQ += dS K_j                          (dS from smem, K_j reused as MN-major B)
//   dkdv: one CTA per 128-key tile; per 128-query tile i (i >= tile):
//           S^T = K Q_i^T, dP^T = V dO_i^T        (tensor core -> TMEM)
//           P^T, dS^T                             (one thread per key row)
//           dV += P^T dO_i, dK += dS^T Q_i        (Q_i / dO_i reused as MN-major B)
// The same smem tile serves as a K-major operand (rows = tokens) and as an
// MN-major operand (K = tokens) — a [128 rows][64 cols] SW128 tile is both
// canonical layouts — so nothing is transposed or loaded twice.
// Warp roles: 0 TMA, 1 MMA (one thread), 2 TMEM alloc, 4..11 math: warp w handles the
// rows of TMEM lane quarter (w-4)%4 and column half (w-4)/4 (no cross-column state
// in the backward, so the per-row work splits freely).
#include "common.cuh"
#include "trace.cuh"
#include "zb_internal.h"

#include <type_traits>

#include <cstdlib>

namespace zb {
namespace fab {

constexpr int T = 128;  // tile rows (queries or keys)
constexpr int kThreads = 384;   // warps 4..11: 8 math warps
constexpr int kMath = 8;        // two per TMEM lane quarter, each on half of the columns
constexpr float LOG2E = 1.4426950408889634f;

ZB_DEVICE uint64_t desc_k(uint32_t base, int kk) {  // K-major [128 rows][64*n] tile
  return umma_desc_sw128(base + (kk >> 2) * T * 128 + (kk & 3) * 32, 16, 1024);
}
ZB_DEVICE uint64_t desc_mn(uint32_t base, int kk) {  // same tile as MN-major, K = rows
  return umma_desc_sw128(base + kk * 2048, T * 128, 1024);
}
// Write 32 consecutive bf16 values (columns c0..c0+31) of row r of a K-major SW128
// [128 rows][128 cols] tile (two 64-col blocks of 16 KB).
ZB_DEVICE void st_row32(uint8_t* tile, int r, int c0, const float* v) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int ch = (c0 >> 3) + q;
    uint4 pk;
    pk.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
    pk.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
    pk.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
    pk.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
    *reinterpret_cast<uint4*>(tile + (ch >> 3) * (T * 128) + r * 128 + (((ch & 7) ^ (r & 7)) << 4)) = pk;
  }
}

// 16 fp32 values of row r, columns [c0, c0+16) (c0 % 16 == 0) -> bf16 into the same
// SWIZZLE_128B tile layout as st_row32.
ZB_DEVICE void st_row16(uint8_t* tile, int r, int c0, const float2 (&v)[8]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int ch = (c0 >> 3) + q;
    uint4 pk;
    pk.x = pack_bf16(v[q * 4 + 0].x, v[q * 4 + 0].y);
    pk.y = pack_bf16(v[q * 4 + 1].x, v[q * 4 + 1].y);
    pk.z = pack_bf16(v[q * 4 + 2].x, v[q * 4 + 2].y);
    pk.w = pack_bf16(v[q * 4 + 3].x, v[q * 4 + 3].y);
    *reinterpret_cast<uint4*>(tile + (ch >> 3) * (T * 128) + r * 128 + (((ch & 7) ^ (r & 7)) << 4)) = pk;
  }
}

// ------------------------------------------------------------------ dQ
template <int D>
struct DqSmem {
  static constexpr int NST = (D == 64) ? 3 : 2;  // K/V stages (192 KB at D = 64, 224 KB at 128)
  static constexpr int DSB = (D == 64) ? 2 : 1;
  static constexpr int TILE = T * D * 2;
  static constexpr int OFF_Q = 0, OFF_DO = TILE;
  static constexpr int OFF_K = 2 * TILE;
  static constexpr int OFF_V = OFF_K + NST * TILE;
  static constexpr int OFF_DS = OFF_V + NST * TILE;
  static constexpr int OFF_BAR = OFF_DS + DSB * T * T * 2;
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    dq_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
              const float* __restrict__ lse, const float* __restrict__ delta,
              __nv_bfloat16* __restrict__ dqkv, int S, int H, int ld, float scale) {
  using L = DqSmem<D>;
  constexpr int NST = L::NST, DSB = L::DSB;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* qo_full = bar;
  uint64_t* kv_full = bar + 1;          // [NST]
  uint64_t* kv_empty = bar + 1 + NST;   // [NST]
  uint64_t* s_full = bar + 1 + 2 * NST;
  uint64_t* s_empty = s_full + 1;
  uint64_t* ds_full = s_full + 2;       // [2]
  uint64_t* ds_empty = s_full + 4;      // [2]
  uint64_t* dq_done = s_full + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 7);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = S / T - 1 - blockIdx.x;
  const int h = blockIdx.y, b = blockIdx.z, HD = H * D, row0 = b * S, nblk = qt + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    mbar_init(qo_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ds_full[i], kMath);
      mbar_init(&ds_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, kMath);
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem, t_dp = tmem + 128, t_dq = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qo_full, 2 * L::TILE);
#pragma unroll
      for (int kc = 0; kc < D / 64; ++kc) {
        tma_load_2d(sm + L::OFF_Q + kc * T * 128, &tm_qkv, qo_full, h * D + kc * 64, row0 + qt * T);
        tma_load_2d(sm + L::OFF_DO + kc * T * 128, &tm_do, qo_full, h * D + kc * 64, row0 + qt * T);
      }
      for (int j = 0; j < nblk; ++j) {
        const int st = j % NST;
        mbar_wait(&kv_empty[st], ((j / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * L::TILE);
#pragma unroll
        for (int kc = 0; kc < D / 64; ++kc) {
          tma_load_2d(sm + L::OFF_K + st * L::TILE + kc * T * 128, &tm_qkv, &kv_full[st],
                      HD + h * D + kc * 64, row0 + j * T);
          tma_load_2d(sm + L::OFF_V + st * L::TILE + kc * T * 128, &tm_qkv, &kv_full[st],
                      2 * HD + h * D + kc * 64, row0 + j * T);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(T, T, 0, 0);
      constexpr uint32_t idesc_q = umma_idesc_bf16(T, D, 0, 1);
      const uint32_t q_base = smem_u32(sm + L::OFF_Q), do_base = smem_u32(sm + L::OFF_DO);
      auto issue_sd = [&](int j) {
        const int st = j % NST;
        mbar_wait(&kv_full[st], (j / NST) & 1);
        mbar_wait(s_empty, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_base = smem_u32(sm + L::OFF_K + st * L::TILE);
        const uint32_t v_base = smem_u32(sm + L::OFF_V + st * L::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          mma_bf16_ss(t_s, desc_k(q_base, kk), desc_k(k_base, kk), idesc_s, kk > 0);
          mma_bf16_ss(t_dp, desc_k(do_base, kk), desc_k(v_base, kk), idesc_s, kk > 0);
        }
        mma_commit(s_full);
      };
      mbar_wait(qo_full, 0);
      tc_fence_after();
      issue_sd(0);
      for (int j = 0; j < nblk; ++j) {
        // With one K/V stage, S_{j+1} must wait for dQ_j to free the stage.
        if (NST > 1 && j + 1 < nblk) issue_sd(j + 1);
        const int st = j % NST, db = j % DSB;
        mbar_wait(&ds_full[db], (j / DSB) & 1);
        tc_fence_after();
        const uint32_t ds_base = smem_u32(sm + L::OFF_DS + db * T * T * 2);
        const uint32_t k_base = smem_u32(sm + L::OFF_K + st * L::TILE);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk)
          mma_bf16_ss(t_dq, desc_k(ds_base, kk), desc_mn(k_base, kk), idesc_q, (j > 0 || kk > 0));
        mma_commit(&kv_empty[st]);
        mma_commit(&ds_empty[db]);
        if (NST == 1 && j + 1 < nblk) issue_sd(j + 1);
      }
      mma_commit(dq_done);
    }
  } else if (warp >= 4) {
    const int wq = (warp - 4) & 3, half = (warp - 4) >> 2, r = wq * 32 + lane, q = qt * T + r;
    const uint32_t lo = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    const size_t vrow = ((size_t)b * H + h) * S + q;
    const float L2 = lse[vrow] * LOG2E, Dl = delta[vrow];
    for (int j = 0; j < nblk; ++j) {
      const int db = j % DSB;
      mbar_wait(&ds_empty[db], ((j / DSB) & 1) ^ 1);
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      uint8_t* ds_tile = sm + L::OFF_DS + db * T * T * 2;
      // dS = P (dP - delta); the causal mask only exists on the diagonal block
      auto chunk = [&](int c, auto diag_c) {
        constexpr bool DG = decltype(diag_c)::value;
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(t_s + lo + c * 32, sv);
        tmem_ld_32x32b_x32(t_dp + lo + c * 32, dv);
        tmem_ld_wait_regs(sv);
        reg_tie(dv);
        float ds[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float p = exp2_fast(fmaf(__uint_as_float(sv[i]), sl2, -L2));
          if (DG && c * 32 + i > r) p = 0.f;
          ds[i] = p * (__uint_as_float(dv[i]) - Dl);
        }
        st_row32(ds_tile, r, c * 32, ds);
      };
      constexpr int CH = T / 64;  // 32-column chunks per half
      if (j == qt) {
#pragma unroll 1
        for (int c = half * CH; c < (half + 1) * CH; ++c) chunk(c, std::true_type{});
      } else {
#pragma unroll 1
        for (int c = half * CH; c < (half + 1) * CH; ++c) chunk(c, std::false_type{});
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ds_full[db]);
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    __nv_bfloat16* out = dqkv + ((size_t)row0 + q) * ld + h * D;
#pragma unroll
    for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_dq + lo + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 pk;
        pk.x = pack_bf16(__uint_as_float(v[i]) * scale, __uint_as_float(v[i + 1]) * scale);
        pk.y = pack_bf16(__uint_as_float(v[i + 2]) * scale, __uint_as_float(v[i + 3]) * scale);
        pk.z = pack_bf16(__uint_as_float(v[i + 4]) * scale, __uint_as_float(v[i + 5]) * scale);
        pk.w = pack_bf16(__uint_as_float(v[i + 6]) * scale, __uint_as_float(v[i + 7]) * scale);
        *reinterpret_cast<uint4*>(out + c * 32 + i) = pk;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------------ dK, dV
template <int D, bool FQ = false>
struct DkvSmem {
  // Q/dO stages (196 KB at D = 64); the fused-dQ variant needs 32 KB of staging
  static constexpr int NST = FQ ? 2 : ((D == 64) ? 3 : 1);
  static constexpr int TILE = T * D * 2;
  static constexpr int OFF_K = 0, OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;              // [NST] Q_i
  static constexpr int OFF_DO = OFF_Q + NST * TILE;   // [NST] dO_i
  static constexpr int OFF_PT = OFF_DO + NST * TILE;  // P^T  [128 keys][128 queries]
  static constexpr int OFF_DST = OFF_PT + T * T * 2;  // dS^T
  static constexpr int OFF_VEC = OFF_DST + T * T * 2; // [2][2][128] fp32 lse*log2e, delta
  static constexpr int OFF_STG = OFF_VEC + 2 * 2 * T * 4;  // FQ: [8 warps] 32x32 fp32
  static constexpr int OFF_BAR = OFF_STG + (FQ ? kMath * 4096 : 0);
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;
};

// FQ (fused dQ, D = 64): the dQ pass is folded into this kernel — per query tile the
// MMA warp also computes the partial dQ_i = dS_i K_kt (A = dS^T tile read as MN-major,
// B = the K tile read as MN-major) into one of two TMEM buffers, and the math warps
// drain it to a fp32 accumulator in global memory with TMA reduce-add stores.  P and
// dS are then computed once instead of twice (the separate dq_kernel recomputes S,
// dP and the exponentials).  The fp32 accumulation order varies between runs.
template <int D, bool FQ = false>
__global__ void __launch_bounds__(kThreads, 1)
    dkdv_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ lse,
                const float* __restrict__ delta, __nv_bfloat16* __restrict__ dqkv, int S, int H,
                int ld, float scale) {
  using L = DkvSmem<D, FQ>;
  constexpr int NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* kv_full = bar;
  uint64_t* qo_full = bar + 1;          // [NST]
  uint64_t* qo_empty = bar + 1 + NST;   // [NST]
  uint64_t* s_full = bar + 1 + 2 * NST;
  uint64_t* s_empty = s_full + 1;
  uint64_t* p_full = s_full + 2;
  uint64_t* p_empty = s_full + 3;
  uint64_t* done = s_full + 4;
  uint64_t* dqp_full = s_full + 5;    // [2] FQ: partial dQ in TMEM
  uint64_t* dqp_empty = s_full + 7;   // [2] FQ: drained by the math warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 9);
  float* vec = reinterpret_cast<float*>(sm + L::OFF_VEC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kt = blockIdx.x;  // early key tiles see the most query tiles: launch first
  const int nqt = S / T;
  const int h = blockIdx.y, b = blockIdx.z, HD = H * D, row0 = b * S;
  const int ntile = nqt - kt;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&qo_full[i], 1);
      mbar_init(&qo_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, kMath);
    mbar_init(p_full, kMath);
    mbar_init(p_empty, 1);
    mbar_init(done, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dqp_full[i], 1);
      mbar_init(&dqp_empty[i], kMath);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_st = tmem, t_dpt = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + D;
  const uint32_t t_dqp = tmem + 256 + 2 * D;  // FQ: [2][D] columns
  griddep_wait();  // PDL: prologue overlapped the previous kernel's tail
  griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * L::TILE);
#pragma unroll
      for (int kc = 0; kc < D / 64; ++kc) {
        tma_load_2d(sm + L::OFF_K + kc * T * 128, &tm_qkv, kv_full, HD + h * D + kc * 64, row0 + kt * T);
        tma_load_2d(sm + L::OFF_V + kc * T * 128, &tm_qkv, kv_full, 2 * HD + h * D + kc * 64,
                    row0 + kt * T);
      }
      for (int i = 0; i < ntile; ++i) {
        const int st = i % NST, qt = kt + i;
        mbar_wait(&qo_empty[st], ((i / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&qo_full[st], 2 * L::TILE);
#pragma unroll
        for (int kc = 0; kc < D / 64; ++kc) {
          tma_load_2d(sm + L::OFF_Q + st * L::TILE + kc * T * 128, &tm_qkv, &qo_full[st],
                      h * D + kc * 64, row0 + qt * T);
          tma_load_2d(sm + L::OFF_DO + st * L::TILE + kc * T * 128, &tm_do, &qo_full[st],
                      h * D + kc * 64, row0 + qt * T);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(T, T, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(T, D, 0, 1);
      const uint32_t k_base = smem_u32(sm + L::OFF_K), v_base = smem_u32(sm + L::OFF_V);
      const uint32_t pt_base = smem_u32(sm + L::OFF_PT), dst_base = smem_u32(sm + L::OFF_DST);
      auto issue_s = [&](int i) {
        const int st = i % NST;
        mbar_wait(&qo_full[st], (i / NST) & 1);
        mbar_wait(s_empty, (i & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sm + L::OFF_Q + st * L::TILE);
        const uint32_t do_base = smem_u32(sm + L::OFF_DO + st * L::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          mma_bf16_ss(t_st, desc_k(k_base, kk), desc_k(q_base, kk), idesc_s, kk > 0);
          mma_bf16_ss(t_dpt, desc_k(v_base, kk), desc_k(do_base, kk), idesc_s, kk > 0);
        }
        mma_commit(s_full);
      };
      mbar_wait(kv_full, 0);
      tc_fence_after();
      issue_s(0);
      for (int i = 0; i < ntile; ++i) {
        if (NST > 1 && i + 1 < ntile) issue_s(i + 1);  // one stage: see dq_kernel
        const int st = i % NST;
        mbar_wait(p_full, i & 1);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sm + L::OFF_Q + st * L::TILE);
        const uint32_t do_base = smem_u32(sm + L::OFF_DO + st * L::TILE);
#pragma unroll
        for (int kk = 0; kk < T / 16; ++kk) {
          mma_bf16_ss(t_dv, desc_k(pt_base, kk), desc_mn(do_base, kk), idesc_o, (i > 0 || kk > 0));
          mma_bf16_ss(t_dk, desc_k(dst_base, kk), desc_mn(q_base, kk), idesc_o, (i > 0 || kk > 0));
        }
        if constexpr (FQ) {  // partial dQ_i = dS_i K (dS^T and K both read as MN-major)
          constexpr uint32_t idesc_q = umma_idesc_bf16(T, D, 1, 1);
          const int bb = i & 1;
          mbar_wait(&dqp_empty[bb], ((i >> 1) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)
            mma_bf16_ss(t_dqp + bb * D, desc_mn(dst_base, kk), desc_mn(k_base, kk), idesc_q,
                        kk > 0 ? 1u : 0u);
          mma_commit(&dqp_full[bb]);
        }
        mma_commit(&qo_empty[st]);
        mma_commit(p_empty);
        if (NST == 1 && i + 1 < ntile) issue_s(i + 1);
      }
      mma_commit(done);
    }
  } else if (warp >= 4) {
    const int wq = (warp - 4) & 3, half = (warp - 4) >> 2, r = wq * 32 + lane;
    const uint32_t lo = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    // FQ: partial dQ of query tile kt+j (this warp: 32 rows x 32 columns) -> fp32
    // accumulator via a TMA reduce-add store from this warp's 4 KB staging area.
    auto drain_dq = [&](int j) {
      uint8_t* stg = sm + L::OFF_STG + (warp - 4) * 4096;
      const int bb = j & 1;
      mbar_wait(&dqp_full[bb], (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(t_dqp + bb * D + lo + half * 32, v);
      tmem_ld_wait_regs(v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&dqp_empty[bb]);
        bulk_wait_read<0>();  // the previous reduce finished reading the staging area
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
            make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                        __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_reduce_add_2d(&tm_dq, stg, h * D + half * 32, row0 + (kt + j) * T + wq * 32);
        bulk_commit();
      }
    };
    const size_t vrow0 = ((size_t)b * H + h) * S + kt * T + r;  // lse / delta one tile ahead
    float nl = 0.f, nd = 0.f;
    if (half == 0) {
      nl = lse[vrow0];
      nd = delta[vrow0];
    }
    for (int i = 0; i < ntile; ++i) {
      const int qt = kt + i;
      float* vl = vec + (i & 1) * 2 * T;
      float* vd = vl + T;
      if (half == 0) {
        vl[r] = nl * LOG2E;
        vd[r] = nd;
        if (i + 1 < ntile) {
          nl = lse[vrow0 + (size_t)(i + 1) * T];
          nd = delta[vrow0 + (size_t)(i + 1) * T];
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the eight math warps
      mbar_wait(s_full, i & 1);
      mbar_wait(p_empty, (i & 1) ^ 1);
      tc_fence_after();
      uint8_t* pt = sm + L::OFF_PT;
      uint8_t* dst = sm + L::OFF_DST;
      // P^T and dS^T rows of this key; the mask only exists on the diagonal tile;
      // the per-query lse / delta come from smem as broadcast 16-byte loads
      auto chunk = [&](int c, auto diag_c) {
        constexpr bool DG = decltype(diag_c)::value;
        uint32_t sv[32], dv[32];
        tmem_ld_32x32b_x32(t_st + lo + c * 32, sv);
        tmem_ld_32x32b_x32(t_dpt + lo + c * 32, dv);
        tmem_ld_wait_regs(sv);
        reg_tie(dv);
        float p[32], ds[32];
#pragma unroll
        for (int t4 = 0; t4 < 32; t4 += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(vl + c * 32 + t4);
          const float4 d4 = *reinterpret_cast<const float4*>(vd + c * 32 + t4);
          const float lv[4] = {l4.x, l4.y, l4.z, l4.w}, dl[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int t = t4 + u;
            float x = exp2_fast(fmaf(__uint_as_float(sv[t]), sl2, -lv[u]));
            if (DG && c * 32 + t < r) x = 0.f;
            p[t] = x;
            ds[t] = x * (__uint_as_float(dv[t]) - dl[u]);
          }
        }
        st_row32(pt, r, c * 32, p);
        st_row32(dst, r, c * 32, ds);
      };
      constexpr int CH = T / 64;  // 32-column chunks per half
      if (qt == kt) {
#pragma unroll 1
        for (int c = half * CH; c < (half + 1) * CH; ++c) chunk(c, std::true_type{});
      } else {
#pragma unroll 1
        for (int c = half * CH; c < (half + 1) * CH; ++c) chunk(c, std::false_type{});
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if constexpr (FQ) {
        if (i > 0) drain_dq(i - 1);
      }
    }
    if constexpr (FQ) {
      drain_dq(ntile - 1);
      if (lane == 0) bulk_wait_all();
    }
    mbar_wait(done, 0);
    tc_fence_after();
    const int k = kt * T + r;
    __nv_bfloat16* dk_row = dqkv + ((size_t)row0 + k) * ld + HD + h * D;
    __nv_bfloat16* dv_row = dk_row + HD;
#pragma unroll
    for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
      uint32_t v[32], w[32];
      tmem_ld_32x32b_x32(t_dk + lo + c * 32, v);
      tmem_ld_32x32b_x32(t_dv + lo + c * 32, w);
      tmem_ld_wait();
#pragma unroll
      for (int t = 0; t < 32; t += 8) {
        uint4 a, bb;
        a.x = pack_bf16(__uint_as_float(v[t]) * scale, __uint_as_float(v[t + 1]) * scale);
        a.y = pack_bf16(__uint_as_float(v[t + 2]) * scale, __uint_as_float(v[t + 3]) * scale);
        a.z = pack_bf16(__uint_as_float(v[t + 4]) * scale, __uint_as_float(v[t + 5]) * scale);
        a.w = pack_bf16(__uint_as_float(v[t + 6]) * scale, __uint_as_float(v[t + 7]) * scale);
        bb.x = pack_bf16(__uint_as_float(w[t]), __uint_as_float(w[t + 1]));
        bb.y = pack_bf16(__uint_as_float(w[t + 2]), __uint_as_float(w[t + 3]));
        bb.z = pack_bf16(__uint_as_float(w[t + 4]), __uint_as_float(w[t + 5]));
        bb.w = pack_bf16(__uint_as_float(w[t + 6]), __uint_as_float(w[t + 7]));
        *reinterpret_cast<uint4*>(dk_row + c * 32 + t) = a;
        *reinterpret_cast<uint4*>(dv_row + c * 32 + t) = bb;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// Persistent fused backward (D = 64): one CTA per SM walks (key tile, head, sequence)
// items heavy-first in boustrophedon order (the one-CTA-per-item grid had 5+ waves of
// CTAs with 1..S/128 query tiles each).  Per item the same pipeline as
// dkdv_kernel<64, true>; barrier parities run on global tile / item counters, the
// Q/dO ring continues across items, and `acc_empty` hands the dK/dV accumulators
// back to the MMA warp once the epilogue read them.
// Shared memory of the persistent fused kernel: P^T lives in TMEM (written over its
// own S^T columns as bf16 and read by the dV MMA as the A operand), which frees the
// room for a DOUBLE-buffered dS^T — the math warps of query tile i+1 no longer wait
// for the dK / dQ MMAs of tile i to finish reading the previous dS^T.
template <int D>
struct DkvqSmem {
  static constexpr int NST = 2;  // Q / dO stages
  static constexpr int TILE = T * D * 2;
  static constexpr int OFF_K = 0, OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;               // [NST] Q_i
  static constexpr int OFF_DO = OFF_Q + NST * TILE;    // [NST] dO_i
  static constexpr int OFF_DST = OFF_DO + NST * TILE;  // [2] dS^T [128 keys][128 queries]
  static constexpr int OFF_VEC = OFF_DST + 2 * T * T * 2;  // [2][2][128] lse*log2e, delta
  static constexpr int OFF_STG = OFF_VEC + 2 * 2 * T * 4;  // [8 warps] 32x32 fp32 dQ staging
  static constexpr int OFF_BAR = OFF_STG + kMath * 4096;
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;
};

// Persistent fused backward (D = 64): one CTA per SM walks (key tile, head, sequence)
// items heavy-first.  Per query tile i of an item the MMA issuer runs
//   dV += P^T(i) dO(i)   [A = P^T from TMEM]     then, in order,
//   S^T(i+1), dP^T(i+1)  [overwrites P^T(i) only after the dV MMA read it]
//   dK += dS^T(i) Q(i),  dQ_i = dS(i) K  [dS^T from the smem buffer of parity i]
// while the math warps turn S^T / dP^T of tile i+1 into P^T (TMEM) and dS^T (the other
// smem buffer) and drain dQ_i (TMA reduce-add into the fp32 accumulator).
template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    dkdvq_persistent_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                            const __grid_constant__ CUtensorMap tm_do,
                            const __grid_constant__ CUtensorMap tm_dq,
                            const float* __restrict__ lse, const float* __restrict__ delta,
                            __nv_bfloat16* __restrict__ dqkv, int S, int H, int n_seq, int ld,
                            float scale) {
  using L = DkvqSmem<D>;
  constexpr int NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* kv_full = bar;
  uint64_t* qo_full = bar + 1;          // [NST]
  uint64_t* qo_empty = bar + 1 + NST;   // [NST]
  uint64_t* s_full = bar + 1 + 2 * NST;
  uint64_t* p_full = s_full + 1;        // P^T (TMEM) and dS^T (smem) of a tile written
  uint64_t* dst_empty = s_full + 2;     // [2] dS^T buffer read by dK / dQ
  uint64_t* done = s_full + 4;          // item's last MMAs complete
  uint64_t* dqp_full = s_full + 5;      // [2]
  uint64_t* dqp_empty = s_full + 7;     // [2]
  uint64_t* kv_empty = s_full + 9;      // item's K / V no longer read
  uint64_t* acc_empty = s_full + 10;    // epilogue read dK / dV (count kMath)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 11);
  float* vec = reinterpret_cast<float*>(sm + L::OFF_VEC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = S / T;
  const int HD = H * D;
  const int per_k = H * n_seq;
  const int items = nqt * per_k;
  const int P = gridDim.x;
  auto item_of = [&](int k) { return k * P + ((k & 1) ? (P - 1 - (int)blockIdx.x) : (int)blockIdx.x); };
  auto decode = [&](int t, int& kt, int& h, int& b) {
    kt = t / per_k;  // key tile 0 sees all nqt query tiles: heaviest first
    const int rem = t % per_k;
    h = rem % H;
    b = rem / H;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&qo_full[i], 1);
      mbar_init(&qo_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, kMath);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dst_empty[i], 1);
      mbar_init(&dqp_full[i], 1);
      mbar_init(&dqp_empty[i], kMath);
    }
    mbar_init(done, 1);
    mbar_init(kv_empty, 1);
    mbar_init(acc_empty, kMath);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_st = tmem, t_dpt = tmem + 128, t_dv = tmem + 256, t_dk = tmem + 256 + D;
  const uint32_t t_dqp = tmem + 256 + 2 * D;
  griddep_wait();
  griddep_launch();
  TR_DECL;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0, lt = 0;
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int kt, h, b;
        decode(t, kt, h, b);
        const int row0 = b * S, ntile = nqt - kt;
        mbar_wait(kv_empty, (lt & 1) ^ 1);
        mbar_arrive_expect_tx(kv_full, 2 * L::TILE);
#pragma unroll
        for (int kc = 0; kc < D / 64; ++kc) {
          tma_load_2d(sm + L::OFF_K + kc * T * 128, &tm_qkv, kv_full, HD + h * D + kc * 64,
                      row0 + kt * T);
          tma_load_2d(sm + L::OFF_V + kc * T * 128, &tm_qkv, kv_full, 2 * HD + h * D + kc * 64,
                      row0 + kt * T);
        }
        for (int i = 0; i < ntile; ++i, ++g) {
          const int st = g % NST, qt = kt + i;
          mbar_wait(&qo_empty[st], ((g / NST) & 1) ^ 1);
          mbar_arrive_expect_tx(&qo_full[st], 2 * L::TILE);
#pragma unroll
          for (int kc = 0; kc < D / 64; ++kc) {
            tma_load_2d(sm + L::OFF_Q + st * L::TILE + kc * T * 128, &tm_qkv, &qo_full[st],
                        h * D + kc * 64, row0 + qt * T);
            tma_load_2d(sm + L::OFF_DO + st * L::TILE + kc * T * 128, &tm_do, &qo_full[st],
                        h * D + kc * 64, row0 + qt * T);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(T, T, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(T, D, 0, 1);
      constexpr uint32_t idesc_q = umma_idesc_bf16(T, D, 1, 1);
      const uint32_t k_base = smem_u32(sm + L::OFF_K), v_base = smem_u32(sm + L::OFF_V);
      int g = 0, lt = 0;
      auto issue_s = [&](int gi) {  // S^T(gi) = K Q^T, dP^T(gi) = V dO^T
        const int st = gi % NST;
        TR_T0();
        mbar_wait(&qo_full[st], (gi / NST) & 1);
        TR_ACC(3);
        tc_fence_after();
        const uint32_t q_base = smem_u32(sm + L::OFF_Q + st * L::TILE);
        const uint32_t do_base = smem_u32(sm + L::OFF_DO + st * L::TILE);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          mma_bf16_ss(t_st, desc_k(k_base, kk), desc_k(q_base, kk), idesc_s, kk > 0);
          mma_bf16_ss(t_dpt, desc_k(v_base, kk), desc_k(do_base, kk), idesc_s, kk > 0);
        }
        mma_commit(s_full);
      };
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int kt, h, b;
        decode(t, kt, h, b);
        const int ntile = nqt - kt;
        mbar_wait(kv_full, lt & 1);
        tc_fence_after();
        issue_s(g);   // the previous item's last dV (reader of P^T in t_st) was issued before
        for (int i = 0; i < ntile; ++i) {
          const int gi = g + i, st = gi % NST, bb = gi & 1;
          TR_T0();
          mbar_wait(p_full, gi & 1);
          TR_ACC(0);
          if (i == 0) mbar_wait(acc_empty, (lt & 1) ^ 1);  // previous item's dK / dV read
          TR_ACC(1);
          tc_fence_after();
          const uint32_t q_base = smem_u32(sm + L::OFF_Q + st * L::TILE);
          const uint32_t do_base = smem_u32(sm + L::OFF_DO + st * L::TILE);
          const uint32_t dst_base = smem_u32(sm + L::OFF_DST + bb * T * T * 2);
          // dV += P^T dO: P^T keys x queries in TMEM; queries [64h, 64h+64) sit in the
          // S^T columns [64h, 64h+32) (each math half wrote its own columns)
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)
            mma_bf16_ts(t_dv, t_st + (kk >> 2) * 64 + (kk & 3) * 8, desc_mn(do_base, kk), idesc_o,
                        (i > 0 || kk > 0) ? 1u : 0u);
          if (i + 1 < ntile) issue_s(gi + 1);  // in order: after the dV MMAs read P^T(i)
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)
            mma_bf16_ss(t_dk, desc_k(dst_base, kk), desc_mn(q_base, kk), idesc_o, (i > 0 || kk > 0));
          TR_T0();
          mbar_wait(&dqp_empty[bb], ((gi >> 1) & 1) ^ 1);
          TR_ACC(2);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < T / 16; ++kk)
            mma_bf16_ss(t_dqp + bb * D, desc_mn(dst_base, kk), desc_mn(k_base, kk), idesc_q,
                        kk > 0 ? 1u : 0u);
          mma_commit(&dqp_full[bb]);
          mma_commit(&qo_empty[st]);
          mma_commit(&dst_empty[bb]);
        }
        mma_commit(kv_empty);
        mma_commit(done);
        g += ntile;
      }
      TR_PRINT("mma", 0);
    }
  } else if (warp >= 4) {
    const int wq = (warp - 4) & 3, half = (warp - 4) >> 2, r = wq * 32 + lane;
    const uint32_t lo = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    int g = 0, lt = 0;
    for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
      int kt, h, b;
      decode(t, kt, h, b);
      const int row0 = b * S, ntile = nqt - kt;
      auto drain_dq = [&](int j) {  // j: tile index within the item
        uint8_t* stg = sm + L::OFF_STG + (warp - 4) * 4096;
        const int gj = g + j, bb = gj & 1;
        TR_T0();
        mbar_wait(&dqp_full[bb], (gj >> 1) & 1);
        tc_fence_after();
        TR_ACC(6);
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_dqp + bb * D + lo + half * 32, v);
        tmem_ld_wait_regs(v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&dqp_empty[bb]);
          bulk_wait_read<0>();
        }
        __syncwarp();
        TR_ACC(7);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
              make_float4(__uint_as_float(v[4 * c]), __uint_as_float(v[4 * c + 1]),
                          __uint_as_float(v[4 * c + 2]), __uint_as_float(v[4 * c + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&tm_dq, stg, h * D + half * 32, row0 + (kt + j) * T + wq * 32);
          bulk_commit();
        }
      };
      // lse / delta of query tile i are loaded from global one tile ahead
      const size_t vrow0 = ((size_t)b * H + h) * S + kt * T + r;
      float nl = 0.f, nd = 0.f;
      if (half == 0) {
        nl = lse[vrow0];
        nd = delta[vrow0];
      }
      for (int i = 0; i < ntile; ++i) {
        const int gi = g + i, qt = kt + i, bb = gi & 1;
        float* vl = vec + bb * 2 * T;
        float* vd = vl + T;
        if (half == 0) {
          vl[r] = nl * LOG2E;
          vd[r] = nd;
          if (i + 1 < ntile) {
            nl = lse[vrow0 + (size_t)(i + 1) * T];
            nd = delta[vrow0 + (size_t)(i + 1) * T];
          }
        }
        TR_T0();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // the eight math warps
        TR_ACC(0);
        mbar_wait(s_full, gi & 1);
        TR_ACC(1);
        mbar_wait(&dst_empty[bb], ((gi >> 1) & 1) ^ 1);  // dK / dQ of tile gi-2 read it
        tc_fence_after();
        TR_ACC(2);
        uint8_t* dst = sm + L::OFF_DST + bb * T * T * 2;
        // The half's 64 S^T / dP^T columns as four 16-column sub-chunks, software-pipelined
        // (the loads of sub-chunk sc+1 are in flight while sc is processed); fp32 pairs
        // go through FFMA2 / FADD2 / FMUL2.
        const uint32_t s_cols = t_st + lo + half * 64, d_cols = t_dpt + lo + half * 64;
        auto sub = [&](auto diag_c, const uint32_t (&sv)[16], const uint32_t (&dv)[16], int sc) {
          constexpr bool DG = decltype(diag_c)::value;
          const int c0 = half * 64 + sc * 16;  // query column of element 0
          float2 ds[8];
          uint32_t pk[8];
#pragma unroll
          for (int t4 = 0; t4 < 16; t4 += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(vl + c0 + t4);
            const float4 d4 = *reinterpret_cast<const float4*>(vd + c0 + t4);
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              const int tt = t4 + u;
              const float2 e = ffma2(make_float2(__uint_as_float(sv[tt]), __uint_as_float(sv[tt + 1])),
                                     make_float2(sl2, sl2),
                                     make_float2(-(u ? l4.z : l4.x), -(u ? l4.w : l4.y)));
              float p0 = exp2_fast(e.x), p1 = exp2_fast(e.y);
              if (DG && c0 + tt < r) p0 = 0.f;
              if (DG && c0 + tt + 1 < r) p1 = 0.f;
              const float2 dd = fadd2(make_float2(__uint_as_float(dv[tt]), __uint_as_float(dv[tt + 1])),
                                      make_float2(-(u ? d4.z : d4.x), -(u ? d4.w : d4.y)));
              ds[tt >> 1] = fmul2(make_float2(p0, p1), dd);
              pk[tt >> 1] = pack_bf16(p0, p1);
            }
          }
          // P^T -> packed TMEM columns inside this half's own (already read) S^T columns
          tmem_st_32x32b_x8(s_cols + sc * 8, pk);
          st_row16(dst, r, c0, ds);
        };
        auto pass = [&](auto diag_c) {
          uint32_t sa[16], da[16], sb[16], db[16];
          tmem_ld_32x32b_x16(s_cols, sa);
          tmem_ld_32x32b_x16(d_cols, da);
          tmem_ld_wait_regs16(sa);
          reg_tie16(da);
#pragma unroll
          for (int sc = 0; sc < 4; sc += 2) {
            tmem_ld_32x32b_x16(s_cols + (sc + 1) * 16, sb);
            tmem_ld_32x32b_x16(d_cols + (sc + 1) * 16, db);
            sub(diag_c, sa, da, sc);
            tmem_ld_wait_regs16(sb);
            reg_tie16(db);
            if (sc + 2 < 4) {
              tmem_ld_32x32b_x16(s_cols + (sc + 2) * 16, sa);
              tmem_ld_32x32b_x16(d_cols + (sc + 2) * 16, da);
            }
            sub(diag_c, sb, db, sc + 1);
            if (sc + 2 < 4) {
              tmem_ld_wait_regs16(sa);
              reg_tie16(da);
            }
          }
        };
        if (qt == kt)
          pass(std::true_type{});
        else
          pass(std::false_type{});
        TR_ACC(3);
        tmem_st_wait();
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        TR_ACC(4);
        if (i > 0) drain_dq(i - 1);
        TR_ACC(5);
        TR_N();
      }
      TR_T0();
      drain_dq(ntile - 1);
      TR_ACC(8);
      mbar_wait(done, lt & 1);
      tc_fence_after();
      TR_ACC(9);
      const int kr = kt * T + r;
      __nv_bfloat16* dk_row = dqkv + ((size_t)row0 + kr) * ld + HD + h * D;
      __nv_bfloat16* dv_row = dk_row + HD;
      // 32-byte stores when every row segment is 32-byte aligned
      const bool st256 = ((reinterpret_cast<uintptr_t>(dqkv) | (ld * 2) | (HD * 2)) & 31) == 0;
#pragma unroll
      for (int c = half * (D / 64); c < (half + 1) * (D / 64); ++c) {
        uint32_t v[32], w[32];
        tmem_ld_32x32b_x32(t_dk + lo + c * 32, v);
        tmem_ld_32x32b_x32(t_dv + lo + c * 32, w);
        tmem_ld_wait_regs(v);
        reg_tie(w);
#pragma unroll
        for (int tt = 0; tt < 32; tt += 16) {
          uint32_t a[8], bq[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            a[e] = pack_bf16(__uint_as_float(v[tt + 2 * e]) * scale,
                             __uint_as_float(v[tt + 2 * e + 1]) * scale);
            bq[e] = pack_bf16(__uint_as_float(w[tt + 2 * e]), __uint_as_float(w[tt + 2 * e + 1]));
          }
          if (st256) {
            st_global_256(dk_row + c * 32 + tt, a);
            st_global_256(dv_row + c * 32 + tt, bq);
          } else {
            *reinterpret_cast<uint4*>(dk_row + c * 32 + tt) = make_uint4(a[0], a[1], a[2], a[3]);
            *reinterpret_cast<uint4*>(dk_row + c * 32 + tt + 8) = make_uint4(a[4], a[5], a[6], a[7]);
            *reinterpret_cast<uint4*>(dv_row + c * 32 + tt) = make_uint4(bq[0], bq[1], bq[2], bq[3]);
            *reinterpret_cast<uint4*>(dv_row + c * 32 + tt + 8) = make_uint4(bq[4], bq[5], bq[6], bq[7]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      TR_ACC(10);
      g += ntile;
    }
    if (lane == 0) bulk_wait_all();
    if (r == 0 && half == 0) TR_PRINT("math", wq);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// delta[b,h,q] = sum_d dO[t,h,d] * O[t,h,d]  (t = b*S + q), and — when dq_accum is
// given — zero that (t, h) slice of the fp32 dQ accumulator in the same pass (it is
// TMA reduce-added into by the fused backward).  D/8 threads per (t, h), one 16-byte
// load of each operand per thread; (t, h) pairs are h-major so the delta writes of a
// warp are contiguous.  Replaces a one-warp-per-row kernel (19 us at GPT-2 small)
// plus a separate memset of the accumulator.
template <int D>
__global__ void __launch_bounds__(256) delta_zero_kernel(const __nv_bfloat16* __restrict__ o,
                                                         const __nv_bfloat16* __restrict__ dout,
                                                         float* __restrict__ delta,
                                                         float* __restrict__ dq_accum, int T,
                                                         int S, int H) {
  pdl_enter();
  constexpr int TPR = D / 8;  // threads per (t, h)
  const int gid = blockIdx.x * (blockDim.x / TPR) + threadIdx.x / TPR;
  const int sub = threadIdx.x % TPR;
  if (gid >= T * H) return;
  const int h = gid / T, t = gid - h * T;
  const size_t off = (size_t)t * H * D + h * D + sub * 8;
  const uint4 a = *reinterpret_cast<const uint4*>(o + off);
  const uint4 g = *reinterpret_cast<const uint4*>(dout + off);
  const uint32_t *ai = &a.x, *gi = &g.x;
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 x = unpack_bf16(ai[k]), y = unpack_bf16(gi[k]);
    acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
  }
#pragma unroll
  for (int m = TPR / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (dq_accum) {
    float4* z = reinterpret_cast<float4*>(dq_accum + off);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (sub == 0) {
    const int b = t / S, q = t - b * S;
    delta[((size_t)b * H + h) * S + q] = acc;
  }
}

// dq (bf16, pitch ld, scaled) = dq_accum (fp32, pitch H*D)
__global__ void dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dqkv,
                                  int rows, int HD, int ld, float scale) {
  pdl_enter();
  const int per_row = HD / 8;
  const int64_t n = (int64_t)rows * per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / per_row), c8 = (int)(i % per_row) * 8;
    const float4 a = *reinterpret_cast<const float4*>(acc + (size_t)row * HD + c8);
    const float4 b = *reinterpret_cast<const float4*>(acc + (size_t)row * HD + c8 + 4);
    uint4 o;
    o.x = pack_bf16(a.x * scale, a.y * scale);
    o.y = pack_bf16(a.z * scale, a.w * scale);
    o.z = pack_bf16(b.x * scale, b.y * scale);
    o.w = pack_bf16(b.z * scale, b.w * scale);
    *reinterpret_cast<uint4*>(dqkv + (size_t)row * ld + c8) = o;
  }
}

template <int D>
static int run(const void* qkv, const void* out, const void* dout, const void* lse, void* dqkv,
               void* dq_accum, void* delta, int n_seq, int S, int H, int ld, float scale,
               cudaStream_t s) {
  const int Tn = n_seq * S;
  const bool fused = D == 64 && dq_accum;
  {
    const int per_cta = 256 / (D / 8);
    cudaError_t e = launch_pdl_k(delta_zero_kernel<D>, dim3((Tn * H + per_cta - 1) / per_cta),
                                 dim3(256), 0, s, (const __nv_bfloat16*)out,
                                 (const __nv_bfloat16*)dout, (float*)delta,
                                 fused ? (float*)dq_accum : (float*)nullptr, Tn, S, H);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd: delta");
  }
  CUtensorMap mq, mo, mdq;
  if (int rc = make_tmap_bf16_2d(&mq, qkv, (uint64_t)3 * H * D, Tn, ld, 64, T)) return rc;
  if (int rc = make_tmap_bf16_2d(&mo, dout, (uint64_t)H * D, Tn, (uint64_t)H * D, 64, T)) return rc;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(dq_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         DqSmem<D>::TOTAL);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(dkdv_kernel<D, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               DkvSmem<D, false>::TOTAL);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd: cudaFuncSetAttribute");
    configured = true;
  }
  const dim3 grid(S / T, H, n_seq);
  if (fused) {
    const int HD = H * D;
    cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)Tn};
    cuuint64_t strides[1] = {(cuuint64_t)HD * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t estr[2] = {1, 1};
    if (int rc = tensor_map_encode(&mdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_accum, dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = DkvqSmem<D>::TOTAL;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool cfg_p = false;
    if (!cfg_p) {
      cudaError_t e0 = cudaFuncSetAttribute(dkdvq_persistent_kernel<D>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            DkvqSmem<D>::TOTAL);
      if (e0 != cudaSuccess) return set_cuda_error(e0, "attn_bwd: cudaFuncSetAttribute");
      cfg_p = true;
    }
    const int items = (S / T) * H * n_seq;
    cfg.gridDim = dim3(items < num_sms() ? items : num_sms());
    cudaError_t e = cudaLaunchKernelEx(&cfg, dkdvq_persistent_kernel<D>, mq, mo, mdq, (const float*)lse,
                                       (const float*)delta, (__nv_bfloat16*)dqkv, S, H, n_seq, ld, scale);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_bwd fused launch");
    const int64_t n8 = (int64_t)Tn * (HD / 8);
    int cg = (int)((n8 + 255) / 256);
    if (cg > num_sms() * 8) cg = num_sms() * 8;
    e = launch_pdl_k(dq_convert_kernel, dim3(cg), dim3(256), 0, s, (const float*)dq_accum,
                     (__nv_bfloat16*)dqkv, Tn, HD, ld, scale);
    return e == cudaSuccess ? 0 : set_cuda_error(e, "attn_bwd fused launch");
  }
  dkdv_kernel<D, false><<<grid, kThreads, DkvSmem<D, false>::TOTAL, s>>>(
        mq, mo, mq /*unused*/, (const float*)lse, (const float*)delta, (__nv_bfloat16*)dqkv, S, H,
        ld, scale);
  dq_kernel<D><<<grid, kThreads, DqSmem<D>::TOTAL, s>>>(mq, mo, (const float*)lse,
                                                        (const float*)delta, (__nv_bfloat16*)dqkv,
                                                        S, H, ld, scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn_bwd launch");
}

}  // namespace fab
}  // namespace zb

using namespace zb;

extern "C" int zb_attn_bwd(const void* qkv, const void* out, const void* dout, const void* lse,
                              void* dqkv, void* dq_accum, void* delta, int n_seq, int S, int H,
                              int D, int ld, float scale, cudaStream_t s) {
  if (S % 128) return set_error(ZB_ERR_INVALID, "attn_bwd: seq_len must be a multiple of 128");
  if (ld % 8 || ((uintptr_t)qkv & 15) || ((uintptr_t)dout & 15))
    return set_error(ZB_ERR_INVALID, "attn_bwd: bad ld/alignment");
  if (n_seq <= 0) return 0;
  if (dq_accum && ((uintptr_t)dq_accum & 15))
    return set_error(ZB_ERR_INVALID, "attn_bwd: dq_accum must be 16-byte aligned");
  if (D == 64)
    return fab::run<64>(qkv, out, dout, lse, dqkv, dq_accum, delta, n_seq, S, H, ld, scale, s);
  if (D == 128)
    return fab::run<128>(qkv, out, dout, lse, dqkv, dq_accum, delta, n_seq, S, H, ld, scale, s);
  return set_error(ZB_ERR_UNSUPPORTED, "attn_bwd: head_dim %d unsupported (64, 128)", D);
}
