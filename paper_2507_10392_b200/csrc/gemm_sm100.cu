// Persistent, warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] = A[M,K] * B[N,K]^T   (bf16 in, fp32 accumulate in TMEM)
//
// A and B may each be K-major (row-major with K contiguous) or MN-major (stored
// [K][M|N], M|N contiguous); the layout is encoded in the TMA box shape, the UMMA
// smem descriptor and the instruction-descriptor major bits, so forward (TN),
// dgrad (B MN-major) and wgrad (A and B MN-major) run through the same pipeline
// without any transpose pass.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = MMA issuer (one thread),
// warp 2 = TMEM allocator, warps 4..11 = epilogue (TMEM -> registers -> global;
// two warps per TMEM lane quarter, each draining half of the tile's columns).
// Work units are (tile, K-split); with split-K (fp32-accumulate epilogue only)
// partial tiles are combined with vectorised fp32 reductions (red.global.add.v4).
// Pipelines: S-stage smem ring (full/empty mbarriers), 2-deep TMEM accumulator
// ring (tmem_full/tmem_empty) so the epilogue of tile i overlaps the mainloop
// of tile i+1. Tiles are BM=128 x BN (128|256), BK=64 (one 128-byte swizzle row).
//
// This is the compute kernel behind the Fwd / Recompute / Bwd tasks the
// reference only models (hetplan simulate.py:330-367, 469-505).
#include "common.cuh"
#include "zb_internal.h"

#include <cstdlib>

namespace zb {

enum Epilogue : int {
  EPI_BF16 = 0,        // C = acc
  EPI_BIAS = 1,        // C = acc + bias[n]
  EPI_BIAS_GELU = 2,   // AUX = acc + bias[n]; C = gelu(AUX)
  EPI_BIAS_RESID = 3,  // C = acc + bias[n] + R[m,n]
  EPI_GELU_BWD = 4,    // C = acc * gelu'(AUX[m,n])
  EPI_F32 = 5,         // C(fp32) = beta * C + acc
  EPI_RESID = 6,       // C = acc + R[m,n]            (bias-free residual, Llama)
};

struct GemmArgs {
  void* C;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* R;  // residual (EPI_BIAS_RESID)
  __nv_bfloat16* aux;      // EPI_BIAS_GELU: written; EPI_GELU_BWD: read
  int M, N, K;
  int ldc, ldr, ldaux;
  float beta;
  int vec;  // 16-byte vector access legal for C / R / aux rows
  int num_m_tiles, num_n_tiles;
  int splits;      // K splits (1 unless EPI_F32 with beta == 1)
  int kb_per_split;
};

constexpr int BM = 128;
// 2-CTA (cta_group::2) tiles are used by default for long-K GEMMs (K >= 2048) whose B
// operand is K-major or whose A is also MN-major (TN, wgrad); dgrad-shaped GEMMs (A
// K-major, B MN-major) measured faster on 1-CTA tiles (profiles/r01_gemm_1cta_vs_2cta.txt).
constexpr bool kPairTilesDefault = true;
constexpr int BK = 64;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 192 ? 5 : 6);
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;  // two accumulators, pow2 alloc
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Apply the epilogue to 32 consecutive accumulator columns of one row and store.
template <int EPI>
ZB_DEVICE void epilogue_chunk(const GemmArgs& args, const uint32_t (&r)[32], int row, int col0) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const bool full = args.vec && (col0 + 32 <= args.N);
  if (EPI == EPI_F32) {
    float* C = reinterpret_cast<float*>(args.C) + (size_t)row * args.ldc + col0;
    if (args.splits > 1) {  // beta == 1: accumulate partial sums in place
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(C + j), "f"(v[j]),
                       "f"(v[j + 1]), "f"(v[j + 2]), "f"(v[j + 3])
                       : "memory");
      } else {
        _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N) atomicAdd(C + j, v[j]);
      }
      return;
    }
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if (args.beta != 0.f) {
          float4 p = *reinterpret_cast<const float4*>(C + j);
          o.x += args.beta * p.x;
          o.y += args.beta * p.y;
          o.z += args.beta * p.z;
          o.w += args.beta * p.w;
        }
        *reinterpret_cast<float4*>(C + j) = o;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N)
        C[j] = v[j] + (args.beta != 0.f ? args.beta * C[j] : 0.f);
    }
    return;
  }
  if (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID) {
    if (full) {
      const uint4* bp = reinterpret_cast<const uint4*>(args.bias + col0);
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        const uint4 q = bp[j / 8];
        float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
               f3 = unpack_bf16(q.w);
        v[j] += f0.x; v[j + 1] += f0.y; v[j + 2] += f1.x; v[j + 3] += f1.y;
        v[j + 4] += f2.x; v[j + 5] += f2.y; v[j + 6] += f3.x; v[j + 7] += f3.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (col0 + j < args.N) v[j] += __bfloat162float(args.bias[col0 + j]);
    }
  }
  if (EPI == EPI_BIAS_RESID || EPI == EPI_RESID) {
    const __nv_bfloat16* Rp = args.R + (size_t)row * args.ldr + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q = *reinterpret_cast<const uint4*>(Rp + j);
        float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
               f3 = unpack_bf16(q.w);
        v[j] += f0.x; v[j + 1] += f0.y; v[j + 2] += f1.x; v[j + 3] += f1.y;
        v[j + 4] += f2.x; v[j + 5] += f2.y; v[j + 6] += f3.x; v[j + 7] += f3.y;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N) v[j] += __bfloat162float(Rp[j]);
    }
  }
  if (EPI == EPI_BIAS_GELU) {
    __nv_bfloat16* Ap = args.aux + (size_t)row * args.ldaux + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q;
        q.x = pack_bf16(v[j], v[j + 1]);
        q.y = pack_bf16(v[j + 2], v[j + 3]);
        q.z = pack_bf16(v[j + 4], v[j + 5]);
        q.w = pack_bf16(v[j + 6], v[j + 7]);
        *reinterpret_cast<uint4*>(Ap + j) = q;
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N) Ap[j] = __float2bfloat16(v[j]);
    }
    // GELU of the bf16-rounded pre-activation, so forward and backward agree.
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(__bfloat162float(__float2bfloat16(v[j])));
  }
  if (EPI == EPI_GELU_BWD) {
    const __nv_bfloat16* Ap = args.aux + (size_t)row * args.ldaux + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q = *reinterpret_cast<const uint4*>(Ap + j);
        float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
               f3 = unpack_bf16(q.w);
        v[j] *= gelu_tanh_grad(f0.x); v[j + 1] *= gelu_tanh_grad(f0.y);
        v[j + 2] *= gelu_tanh_grad(f1.x); v[j + 3] *= gelu_tanh_grad(f1.y);
        v[j + 4] *= gelu_tanh_grad(f2.x); v[j + 5] *= gelu_tanh_grad(f2.y);
        v[j + 6] *= gelu_tanh_grad(f3.x); v[j + 7] *= gelu_tanh_grad(f3.y);
      }
    } else {
      _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N)
        v[j] *= gelu_tanh_grad(__bfloat162float(Ap[j]));
    }
  }
  __nv_bfloat16* Cp = reinterpret_cast<__nv_bfloat16*>(args.C) + (size_t)row * args.ldc + col0;
  if (full) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 q;
      q.x = pack_bf16(v[j], v[j + 1]);
      q.y = pack_bf16(v[j + 2], v[j + 3]);
      q.z = pack_bf16(v[j + 4], v[j + 5]);
      q.w = pack_bf16(v[j + 6], v[j + 7]);
      *reinterpret_cast<uint4*>(Cp + j) = q;
    }
  } else {
    _Pragma("unroll") for (int j = 0; j < 32; ++j) if (col0 + j < args.N) Cp[j] = __float2bfloat16(v[j]);
  }
}

template <int BN, int A_MN, int B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B atoms.
  uint32_t base = smem_u32(smem_raw);
  uint32_t pad = ((base + 1023u) & ~1023u) - base;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smA = smem;
  uint8_t* smB = smem + S * Cfg::A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = args.num_m_tiles * args.num_n_tiles;
  const int num_units = num_tiles * args.splits;
  const int num_kb = (args.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], kEpiWarps);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        const int m0 = (tile % args.num_m_tiles) * BM;
        const int n0 = (tile / args.num_m_tiles) * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          uint8_t* a_dst = smA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = smB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(a_dst + j * (64 * BK * 2), &tmA, &full_bar[stage], m0 + j * 64, k0);
          } else {
            tma_load_2d(a_dst, &tmA, &full_bar[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(b_dst + j * (64 * BK * 2), &tmB, &full_bar[stage], n0 + j * 64, k0);
          } else {
            tma_load_2d(b_dst, &tmB, &full_bar[stage], k0, n0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(smB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: 8-row groups 1024 B apart, advance 32 B per K=16 step.
            // MN-major: 64-wide MN chunks BK*128 B apart (LBO), 8-row K groups
            //           1024 B apart (SBO), advance 16 rows = 2048 B per K step.
            uint64_t a_desc = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                   : umma_desc_sw128(a_addr + k * 32, 16, 1024);
            uint64_t b_desc = B_MN ? umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024)
                                   : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_bf16_ss(d_tmem, a_desc, b_desc, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          mma_commit(&empty_bar[stage]);  // smem slot free once these MMAs retire
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int ew = (warp - 4) & 3;     // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;  // which half of the tile's columns it drains
    int local = 0;
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
      const int tile = unit % num_tiles;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % args.num_m_tiles) * BM;
      const int n0 = (tile / args.num_m_tiles) * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const bool row_ok = row < args.M;
#pragma unroll 1
      for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
        __syncwarp();
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int col0 = n0 + c * 32;
        if (row_ok && col0 < args.N) epilogue_chunk<EPI>(args, r, row, col0);
      }
      // Accumulator drained: hand it back to the MMA warp.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
}

// ---------------------------------------------------------------- 2-CTA variant
// A CTA pair (cluster of 2, cta_group::2) computes a 256 x BN tile: each CTA
// stages its 128 rows of A and half of B's BN columns, the leader CTA's single
// thread issues tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem, and
// each CTA's TMEM receives its own 128 accumulator rows.  Per SM the smem
// operand traffic per MMA cycle drops by a third vs. the 1-CTA 128 x 256 tile.
template <int BN>
struct Gemm2Cfg {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 6 : (BN == 192 ? 7 : 8);
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, int A_MN, int B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm2cta_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB, GemmArgs args) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int S = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base + 1023u) & ~1023u) - base);
  uint8_t* smA = smem;
  uint8_t* smB = smem + S * Cfg::A_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int num_tiles = args.num_m_tiles * args.num_n_tiles;  // m tiles of 256 rows
  const int num_units = num_tiles * args.splits;
  const int num_kb = (args.K + BK - 1) / BK;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);   // leader's expect_tx (both CTAs' TMA bytes land here)
      mbar_init(&empty_bar[i], 1);  // multicast MMA commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiWarps);  // both CTAs' epilogue warps (leader's copy)
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2cta(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = cluster; unit < num_units; unit += nclusters) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        const int m0 = (tile % args.num_m_tiles) * 256 + (int)rank * 128;
        const int n0 = (tile / args.num_m_tiles) * BN + (int)rank * (BN / 2);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          // Only the leader arrives (with both CTAs' bytes).  The follower's TMA
          // bytes for this phase cannot land early: it refills a stage only after the
          // pair's MMA released it, i.e. after the leader's barrier completed the
          // previous phase.  (A remote release-arrive per k-block costs a MEMBAR.)
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::STAGE_BYTES);
          uint8_t* a_dst = smA + stage * Cfg::A_BYTES;
          uint8_t* b_dst = smB + stage * Cfg::B_BYTES;
          const int k0 = kb * BK;
          if (A_MN) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              tma_load_2d_2cta(a_dst + j * (64 * BK * 2), &tmA, &full_bar[stage], m0 + j * 64, k0);
          } else {
            tma_load_2d_2cta(a_dst, &tmA, &full_bar[stage], k0, m0);
          }
          if (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 128; ++j)
              tma_load_2d_2cta(b_dst + j * (64 * BK * 2), &tmB, &full_bar[stage], n0 + j * 64, k0);
          } else {
            tma_load_2d_2cta(b_dst, &tmB, &full_bar[stage], k0, n0);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(256, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int unit = cluster; unit < num_units; unit += nclusters, ++local) {
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smA + stage * Cfg::A_BYTES);
          const uint32_t b_addr = smem_u32(smB + stage * Cfg::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t a_desc = A_MN ? umma_desc_sw128(a_addr + k * 2048, BK * 128, 1024)
                                   : umma_desc_sw128(a_addr + k * 32, 16, 1024);
            uint64_t b_desc = B_MN ? umma_desc_sw128(b_addr + k * 2048, BK * 128, 1024)
                                   : umma_desc_sw128(b_addr + k * 32, 16, 1024);
            mma_bf16_ss_2cta(d_tmem, a_desc, b_desc, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          mma_commit_2cta(&empty_bar[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2cta(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    const int ew = (warp - 4) & 3;
    const int half = (warp - 4) >> 2;
    int local = 0;
    for (int unit = cluster; unit < num_units; unit += nclusters, ++local) {
      const int tile = unit % num_tiles;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile % args.num_m_tiles) * 256 + (int)rank * 128;
      const int n0 = (tile / args.num_m_tiles) * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const bool row_ok = row < args.M;
#pragma unroll 1
      for (int c = half * (BN / 64); c < (half + 1) * (BN / 64); ++c) {
        __syncwarp();
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, r);
        tmem_ld_wait();
        const int col0 = n0 + c * 32;
        if (row_ok && col0 < args.N) epilogue_chunk<EPI>(args, r, row, col0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tempty_bar[acc]);
        else
          mbar_arrive_remote(&tempty_bar[acc], 0);
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2cta(tmem_base, Cfg::TMEM_COLS);
}

// ---------------------------------------------------------------- host side

// 2-D bf16 tensor map with a {64, rows} box and 128-byte swizzle.
// inner = contiguous extent (elements), outer = number of rows, ld = row pitch (elements).
static int make_tmap(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  return tensor_map_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

template <int BN, int A_MN, int B_MN, int EPI>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs args,
                       cudaStream_t stream) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_sm100_kernel<BN, A_MN, B_MN, EPI>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm: cudaFuncSetAttribute");
    configured = true;
  }
  args.num_m_tiles = (args.M + BM - 1) / BM;
  args.num_n_tiles = (args.N + BN - 1) / BN;
  const int tiles = args.num_m_tiles * args.num_n_tiles;
  const int num_kb = (args.K + BK - 1) / BK;
  int splits = 1;
  if (EPI == EPI_F32 && args.beta == 1.f && tiles < num_sms()) {
    // split K so that at least ~2 waves of (tile, split) units exist, >= 8 k-blocks each
    splits = (2 * num_sms() + tiles - 1) / tiles;
    int cap = num_kb / 8;
    if (splits > cap) splits = cap > 1 ? cap : 1;
  }
  args.kb_per_split = (num_kb + splits - 1) / splits;
  args.splits = (num_kb + args.kb_per_split - 1) / args.kb_per_split;
  const int units = tiles * args.splits;
  int grid = units < num_sms() ? units : num_sms();
  kern<<<grid, kThreads, Cfg::SMEM_BYTES, stream>>>(ta, tb, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  return 0;
}

template <int BN, int A_MN, int B_MN, int EPI>
static int launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs args,
                        cudaStream_t stream) {
  using Cfg = Gemm2Cfg<BN>;
  auto kern = gemm2cta_kernel<BN, A_MN, B_MN, EPI>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm2cta: cudaFuncSetAttribute");
    configured = true;
  }
  args.num_m_tiles = (args.M + 255) / 256;
  args.num_n_tiles = (args.N + BN - 1) / BN;
  const int tiles = args.num_m_tiles * args.num_n_tiles;
  const int num_kb = (args.K + BK - 1) / BK;
  const int pairs = num_sms() / 2;
  int splits = 1;
  if (EPI == EPI_F32 && args.beta == 1.f && tiles < pairs) {
    splits = (2 * pairs + tiles - 1) / tiles;
    int cap = num_kb / 8;
    if (splits > cap) splits = cap > 1 ? cap : 1;
  }
  args.kb_per_split = (num_kb + splits - 1) / splits;
  args.splits = (num_kb + args.kb_per_split - 1) / args.kb_per_split;
  const int units = tiles * args.splits;
  const int clusters = units < pairs ? units : pairs;
  kern<<<2 * clusters, kThreads, Cfg::SMEM_BYTES, stream>>>(ta, tb, args);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "gemm2cta launch");
  return 0;
}

template <int BN, int A_MN, int B_MN>
static int dispatch_epi2(int epi, const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs args,
                         cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch_gemm2<BN, A_MN, B_MN, EPI_BF16>(ta, tb, args, s);
    case EPI_BIAS: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS>(ta, tb, args, s);
    case EPI_BIAS_GELU: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS_GELU>(ta, tb, args, s);
    case EPI_BIAS_RESID: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS_RESID>(ta, tb, args, s);
    case EPI_GELU_BWD: return launch_gemm2<BN, A_MN, B_MN, EPI_GELU_BWD>(ta, tb, args, s);
    case EPI_F32: return launch_gemm2<BN, A_MN, B_MN, EPI_F32>(ta, tb, args, s);
    case EPI_RESID: return launch_gemm2<BN, A_MN, B_MN, EPI_RESID>(ta, tb, args, s);
  }
  return set_error(ZB_ERR_INVALID, "gemm: unknown epilogue %d", epi);
}

template <int BN, int A_MN, int B_MN>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, GemmArgs args,
                        cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch_gemm<BN, A_MN, B_MN, EPI_BF16>(ta, tb, args, s);
    case EPI_BIAS: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS>(ta, tb, args, s);
    case EPI_BIAS_GELU: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS_GELU>(ta, tb, args, s);
    case EPI_BIAS_RESID: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS_RESID>(ta, tb, args, s);
    case EPI_GELU_BWD: return launch_gemm<BN, A_MN, B_MN, EPI_GELU_BWD>(ta, tb, args, s);
    case EPI_F32: return launch_gemm<BN, A_MN, B_MN, EPI_F32>(ta, tb, args, s);
    case EPI_RESID: return launch_gemm<BN, A_MN, B_MN, EPI_RESID>(ta, tb, args, s);
  }
  return set_error(ZB_ERR_INVALID, "gemm: unknown epilogue %d", epi);
}

}  // namespace zb

using namespace zb;

extern "C" int zb_gemm_bf16(const void* A, const void* B, void* C, const void* bias,
                            const void* R, void* aux, int M, int N, int K, int lda, int ldb,
                            int ldc, int ldr, int ldaux, int a_mn_major, int b_mn_major,
                            int epilogue, float beta, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(ZB_ERR_INVALID, "gemm: bad shape %d %d %d", M, N, K);
  if ((lda % 8) || (ldb % 8))
    return set_error(ZB_ERR_INVALID, "gemm: lda/ldb must be multiples of 8 elements");
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15))
    return set_error(ZB_ERR_INVALID, "gemm: A/B must be 16-byte aligned");
  CUtensorMap ta, tb;
  // Tile choice by a wave-quantisation cost model: cost = waves x per-tile time per
  // k-block on one SM = max(MMA 2*BN cycles, smem operand bytes at ~87% of 128 B/cycle).
  // 1-CTA tiles are 128 x BN on one SM; 2-CTA (cta_group::2) tiles are 256 x BN on an
  // SM pair, each SM staging 128 rows of A and BN/2 rows of B.
  int BN = 256, pair = 0;
  {
    static int force = -1;  // ZB_GEMM_CTAS=1|2 pins 1-CTA / 2-CTA tiles (benchmarking)
    if (force < 0) {
      const char* f = getenv("ZB_GEMM_CTAS");
      force = f ? atoi(f) : 0;
    }
    const bool shape_ok = K >= 2048 && !(b_mn_major && !a_mn_major);
    const bool allow_pair = force == 2 || (kPairTilesDefault && force != 1 && shape_ok);
    const int sms = num_sms();
    double best = 1e30;
    for (int two = 1; two >= 0; --two) {
      if (two && (M < 256 || !allow_pair)) continue;
      if (!two && force == 2 && M >= 256) continue;
      for (int bn : {256, 192, 128}) {
        if (two && b_mn_major && bn == 192) continue;  // MN-major half-tiles must be 64-multiples
        const long long t = (long long)((M + (two ? 255 : 127)) / (two ? 256 : 128)) * ((N + bn - 1) / bn);
        const long long slots = two ? sms / 2 : sms;
        const long long waves = (t + slots - 1) / slots;
        const double smem_cyc = 1.15 * (128 + (two ? bn / 2 : bn));
        const double per = 2.0 * bn > smem_cyc ? 2.0 * bn : smem_cyc;
        const double cost = waves * per;
        if (cost < best - 1e-9) {
          best = cost;
          BN = bn;
          pair = two;
        }
      }
    }
    if (N <= 128) BN = 128;
  }
  int rc;
  if (a_mn_major)
    rc = make_tmap(&ta, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, BK);
  else
    rc = make_tmap(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BM);
  if (rc) return rc;
  if (b_mn_major)
    rc = make_tmap(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, BK);
  else
    rc = make_tmap(&tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, (uint32_t)(pair ? BN / 2 : BN));
  if (rc) return rc;
  GemmArgs args{};
  args.C = C;
  args.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
  args.R = reinterpret_cast<const __nv_bfloat16*>(R);
  args.aux = reinterpret_cast<__nv_bfloat16*>(aux);
  args.M = M; args.N = N; args.K = K;
  args.ldc = ldc; args.ldr = ldr; args.ldaux = ldaux;
  args.beta = beta;
  {
    const int celem = (epilogue == EPI_F32) ? 4 : 8;  // elements per 16 bytes
    bool v = (ldc % celem) == 0 && ((uintptr_t)C & 15) == 0;
    if (R) v = v && (ldr % 8) == 0 && ((uintptr_t)R & 15) == 0;
    if (aux) v = v && (ldaux % 8) == 0 && ((uintptr_t)aux & 15) == 0;
    if (bias) v = v && ((uintptr_t)bias & 15) == 0;
    args.vec = v ? 1 : 0;
  }
  const int key = a_mn_major * 2 + b_mn_major;
  if (pair) {
    if (BN == 256) {
      switch (key) {
        case 0: return dispatch_epi2<256, 0, 0>(epilogue, ta, tb, args, stream);
        case 1: return dispatch_epi2<256, 0, 1>(epilogue, ta, tb, args, stream);
        case 3: return dispatch_epi2<256, 1, 1>(epilogue, ta, tb, args, stream);
      }
    } else if (BN == 192) {
      switch (key) {
        case 0: return dispatch_epi2<192, 0, 0>(epilogue, ta, tb, args, stream);
      }
    } else {
      switch (key) {
        case 0: return dispatch_epi2<128, 0, 0>(epilogue, ta, tb, args, stream);
        case 1: return dispatch_epi2<128, 0, 1>(epilogue, ta, tb, args, stream);
        case 3: return dispatch_epi2<128, 1, 1>(epilogue, ta, tb, args, stream);
      }
    }
    return set_error(ZB_ERR_INVALID, "gemm: unsupported 2-CTA layout");
  }
  if (BN == 256) {
    switch (key) {
      case 0: return dispatch_epi<256, 0, 0>(epilogue, ta, tb, args, stream);
      case 1: return dispatch_epi<256, 0, 1>(epilogue, ta, tb, args, stream);
      case 3: return dispatch_epi<256, 1, 1>(epilogue, ta, tb, args, stream);
    }
  } else if (BN == 192) {
    switch (key) {
      case 0: return dispatch_epi<192, 0, 0>(epilogue, ta, tb, args, stream);
      case 1: return dispatch_epi<192, 0, 1>(epilogue, ta, tb, args, stream);
      case 3: return dispatch_epi<192, 1, 1>(epilogue, ta, tb, args, stream);
    }
  } else {
    switch (key) {
      case 0: return dispatch_epi<128, 0, 0>(epilogue, ta, tb, args, stream);
      case 1: return dispatch_epi<128, 0, 1>(epilogue, ta, tb, args, stream);
      case 3: return dispatch_epi<128, 1, 1>(epilogue, ta, tb, args, stream);
    }
  }
  return set_error(ZB_ERR_INVALID, "gemm: unsupported layout (A MN-major with B K-major)");
}
