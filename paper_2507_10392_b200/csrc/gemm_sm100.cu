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
// Roles (128 + 32 * kEpiWarps threads): warp 0 = TMA producer, warp 1 = MMA issuer (one
// thread), warp 2 = TMEM allocator, warps 4.. = epilogue (TMEM -> registers -> global;
// kEpiWarps / 4 warps per TMEM lane quarter, each draining a run of the tile's columns).
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

#ifndef ZB_GEMM_EXP
#define ZB_GEMM_EXP 0  // 0 = product; 1/2/3 = timing experiments (separate builds)
#endif

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <dlfcn.h>
#include <vector>
#include <tuple>
#include <mutex>
#include <map>

namespace zb {

enum Epilogue : int {
  EPI_BF16 = 0,        // C = acc
  EPI_BIAS = 1,        // C = acc + bias[n]
  EPI_BIAS_GELU = 2,   // AUX = acc + bias[n]; C = gelu(AUX)
  EPI_BIAS_RESID = 3,  // C = acc + bias[n] + R[m,n]
  EPI_GELU_BWD = 4,    // C = acc * gelu'(AUX[m,n])
  EPI_F32 = 5,         // C(fp32) = beta * C + acc
  EPI_RESID = 6,       // C = acc + R[m,n]            (bias-free residual, Llama)
  EPI_BIAS_GELU_NA = 7,  // C = gelu(acc + bias), pre-activation not kept (forward pass)
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
  int tma_epi;     // 1: TMA-store epilogue (aligned C / R / aux, beta in {0, 1})
  int n_fastest;   // tile raster: 1 = consecutive units walk N (A panel read once)
};

// Tile raster.  M-fastest (default): the CTAs in flight share B column panels and
// sweep all of A, which must stay L2-resident between n-columns.  N-fastest: the
// CTAs in flight cover every n-tile of a few A row panels, so A streams from HBM
// once and B must stay resident — chosen when A is the larger operand and does not
// fit in L2 (LM-head dgrad / wgrad: A = the [tokens, vocab] logits gradient, 824 MB
// at GPT-2 small, read 3-4x from HBM under the M-fastest raster).
__device__ __forceinline__ void tile_mn(const GemmArgs& a, int tile, int& mt, int& nt) {
  if (a.n_fastest) {
    nt = tile % a.num_n_tiles;
    mt = tile / a.num_n_tiles;
  } else {
    mt = tile % a.num_m_tiles;
    nt = tile / a.num_m_tiles;
  }
}

constexpr int BM = 128;
// 2-CTA (cta_group::2) tiles are used by default for long-K GEMMs (K >= 2048) whose B
// operand is K-major or whose A is also MN-major (TN, wgrad); dgrad-shaped GEMMs (A
// K-major, B MN-major) measured faster on 1-CTA tiles (profiles/r01_gemm_1cta_vs_2cta.txt).
constexpr bool kPairTilesDefault = true;
constexpr int BK = 64;
#ifndef ZB_EPI_WARPS
#define ZB_EPI_WARPS 8
#endif
// Epilogue warps: kEpiWarps / 4 per TMEM lane quarter, each draining a contiguous run
// of the tile's 32-column chunks (the K = 768 GEMMs of the step are bound by the
// per-chunk epilogue chain, so more warps per quarter = more chains in flight).
constexpr int kEpiWarps = ZB_EPI_WARPS;
static_assert(kEpiWarps % 4 == 0, "epilogue warps come in lane-quarter groups");
constexpr int kEpiParts = kEpiWarps / 4;
constexpr int kThreads = 128 + 32 * kEpiWarps;
constexpr int kSmemMax = 232448;  // max dynamic shared memory per block (227 KB)
// Chunk range [cb, ce) of epilogue part p for a tile of `nch` 32-column chunks.
__host__ __device__ constexpr int epi_cb(int p, int nch) { return p * nch / kEpiParts; }

// Epilogue staging slots (2 KB each) per epilogue warp: 4 when the smem budget holds
// them without losing a pipeline stage or still leaves >= 6 stages (the TMA stores of
// up to three earlier chunks then stay in flight), else 2.
constexpr int epi_slots(int stage_bytes) {
  return ((kSmemMax - 1536 - kEpiWarps * 8192) / stage_bytes ==
              (kSmemMax - 1536 - kEpiWarps * 4096) / stage_bytes ||
          (kSmemMax - 1536 - kEpiWarps * 8192) / stage_bytes >= 6)
             ? 4 : 2;
}

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int NS = epi_slots(STAGE_BYTES);
  static constexpr int EPI_BYTES = kEpiWarps * NS * 2048;  // per-epilogue-warp TMA staging
  static constexpr int FIT = (kSmemMax - 1536 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = FIT < 8 ? FIT : 8;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;  // two accumulators, pow2 alloc
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 512 /*barriers*/;
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
  if (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID || EPI == EPI_BIAS_GELU_NA) {
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
    gelu32_bf16in(v);   // GELU of the bf16-rounded pre-activation, so forward and backward agree
  }
  if (EPI == EPI_BIAS_GELU_NA) gelu32_bf16in(v);
  if (EPI == EPI_GELU_BWD) {
    const __nv_bfloat16* Ap = args.aux + (size_t)row * args.ldaux + col0;
    if (full) {
#pragma unroll
      float in[32];
      for (int j = 0; j < 32; j += 8) {
        uint4 q = *reinterpret_cast<const uint4*>(Ap + j);
        float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z),
               f3 = unpack_bf16(q.w);
        in[j] = f0.x; in[j + 1] = f0.y; in[j + 2] = f1.x; in[j + 3] = f1.y;
        in[j + 4] = f2.x; in[j + 5] = f2.y; in[j + 6] = f3.x; in[j + 7] = f3.y;
      }
      gelu_grad_mul32(v, in);
    } else {
      float in[32];
      _Pragma("unroll") for (int j = 0; j < 32; ++j)
        in[j] = col0 + j < args.N ? __bfloat162float(Ap[j]) : 0.f;
      gelu_grad_mul32(v, in);
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

// ---------------------------------------------------------------- TMA epilogue
// Each epilogue warp owns a 32-row slab of the tile and drains it in 32-column
// chunks through a 4 KB shared staging area (two 2 KB slots): the thread of row r
// writes its 64-byte (bf16) or 128-byte (fp32) row of the chunk into the slot in
// the TMA swizzle layout (conflict-free), and one lane issues a TMA tile store —
// or, for fp32 accumulation (beta = 1 / split-K), a TMA reduce-add store — so the
// global writes leave the SM as full lines instead of 32 row-strided 16-byte
// pieces per instruction.  Residual / GELU-backward operands are TMA-loaded into
// the slot (prefetched one chunk ahead) and read back from shared memory.
constexpr int kEpiSlot = 2048;

struct EpiMaps {
  const CUtensorMap* C;
  const CUtensorMap* aux;
  const CUtensorMap* R;
};

// byte offset of 16-byte chunk j of row r in a [32 rows][64 B] SWIZZLE_64B box
ZB_DEVICE uint32_t sw64(int r, int j) { return r * 64 + ((j ^ ((r >> 1) & 3)) << 4); }
// ... and in a [32 rows][128 B] SWIZZLE_128B box
ZB_DEVICE uint32_t sw128(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

ZB_DEVICE void st_row_bf16(uint8_t* slot, int r, const float (&v)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 q;
    q.x = pack_bf16(v[8 * j], v[8 * j + 1]);
    q.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
    q.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
    q.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
    *reinterpret_cast<uint4*>(slot + sw64(r, j)) = q;
  }
}

ZB_DEVICE void ld_row_bf16(const uint8_t* slot, int r, float (&o)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 q = *reinterpret_cast<const uint4*>(slot + sw64(r, j));
    float2 f0 = unpack_bf16(q.x), f1 = unpack_bf16(q.y), f2 = unpack_bf16(q.z), f3 = unpack_bf16(q.w);
    o[8 * j] = f0.x; o[8 * j + 1] = f0.y; o[8 * j + 2] = f1.x; o[8 * j + 3] = f1.y;
    o[8 * j + 4] = f2.x; o[8 * j + 5] = f2.y; o[8 * j + 6] = f3.x; o[8 * j + 7] = f3.y;
  }
}

// Drain one accumulator slab.  tacc = TMEM address of column 0 of this warp's lane
// quarter in the accumulator; chunks [cb, ce) of 32 columns; row0 / n0 = global
// coordinates of the slab's first row / the tile's first column.  `release` is
// called once the last TMEM read retired (the accumulator may be reused).
template <int EPI, int NS, typename Release>
ZB_DEVICE void epilogue_tma(const GemmArgs& args, const EpiMaps& maps, uint8_t* stg,
                            uint64_t* ebar, uint32_t& eph, uint32_t& ecnt, uint32_t tacc,
                            uint64_t* tfull,
                            uint32_t tfull_parity, int row0, int n0, int cb, int ce, int lane,
                            Release release) {
  constexpr bool LOADS = (EPI == EPI_BIAS_RESID || EPI == EPI_RESID || EPI == EPI_GELU_BWD);
  const CUtensorMap* tm_in = EPI == EPI_GELU_BWD ? maps.aux : maps.R;
  // Prefetch the first chunk's residual / aux operand before the accumulator is ready.
  if (LOADS) {
    if (lane == 0) {
      bulk_wait_read<0>();
      mbar_arrive_expect_tx(&ebar[0], kEpiSlot);
      tma_load_2d(stg, tm_in, &ebar[0], n0 + cb * 32, row0);
    }
  }
  constexpr bool BIAS = (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_BIAS_RESID ||
                         EPI == EPI_BIAS_GELU_NA);
  // Bias vectors of a chunk (same for every row) are loaded one chunk ahead, so the
  // global-load latency never sits on the chunk's critical path.
  auto load_bias = [&](int c, uint4 (&q)[4]) {
    const int col = n0 + c * 32;
    if (col + 32 <= args.N) {
      const uint4* bp = reinterpret_cast<const uint4*>(args.bias + col);
#pragma unroll
      for (int j = 0; j < 4; ++j) q[j] = bp[j];
    }
  };
  uint4 bq[4];
  if (BIAS) load_bias(cb, bq);
  mbar_wait(tfull, tfull_parity);
  tc_fence_after();
#pragma unroll 1
  for (int c = cb; c < ce; ++c) {
    const int k = c - cb;
    const int col0 = n0 + c * 32;
    uint8_t* slot = stg + (k & 1) * kEpiSlot;  // LOADS path: per-tile slot order
    if (LOADS && c + 1 < ce && lane == 0) {  // prefetch the next chunk into the other slot
      bulk_wait_read<0>();
      const int ns = (k + 1) & 1;
      mbar_arrive_expect_tx(&ebar[ns], kEpiSlot);
      tma_load_2d(stg + ns * kEpiSlot, tm_in, &ebar[ns], col0 + 32, row0);
    }
    uint4 bn[4];
    if (BIAS && c + 1 < ce) load_bias(c + 1, bn);
    __syncwarp();
    uint32_t r[32];
    tmem_ld_32x32b_x32(tacc + c * 32, r);
    tmem_ld_wait_regs(r);
    if (c + 1 == ce) {
      tc_fence_before();
      __syncwarp();
      release();
    }
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    if (BIAS) {
      if (col0 + 32 <= args.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          const uint4 q = bq[j / 8];
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
    if (LOADS) {
      const int bs = k & 1;
      mbar_wait(&ebar[bs], (eph >> bs) & 1);
      eph ^= 1u << bs;
      float in[32];
      ld_row_bf16(slot, lane, in);
      if (EPI == EPI_GELU_BWD) {
        gelu_grad_mul32(v, in);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += in[j];
      }
      st_row_bf16(slot, lane, v);   // in place: each thread rewrites only its own row
    } else if (EPI == EPI_F32) {
      // one 4 KB slot per chunk; with NS = 4 two of them alternate (the slot written
      // now was last stored two chunks ago)
      slot = stg + (NS == 4 ? (ecnt & 1) * 2 * kEpiSlot : 0);
      ++ecnt;
      if (lane == 0) {
        if (NS == 4) bulk_wait_read<1>(); else bulk_wait_read<0>();
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(slot + sw128(lane, j)) =
            make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else if (EPI == EPI_BIAS_GELU) {
      // aux -> even slot, C -> odd slot of a pair; with NS = 4 two pairs alternate
      slot = stg + (NS == 4 ? (ecnt & 1) * 2 * kEpiSlot : 0);
      ++ecnt;
      if (lane == 0) {
        if (NS == 4) bulk_wait_read<1>(); else bulk_wait_read<0>();
      }
      __syncwarp();
      st_row_bf16(slot, lane, v);
      gelu32_bf16in(v);   // GELU of the bf16-rounded pre-activation (= the stored aux)
      st_row_bf16(slot + kEpiSlot, lane, v);
    } else {
      if (EPI == EPI_BIAS_GELU_NA) gelu32_bf16in(v);
      // slots rotate over a running chunk count (across tiles), so the slot written
      // now was last stored NS chunks ago
      slot = stg + (ecnt % NS) * kEpiSlot;
      ++ecnt;
      if (lane == 0) {
        if (NS == 4) bulk_wait_read<3>(); else bulk_wait_read<1>();
      }
      __syncwarp();
      st_row_bf16(slot, lane, v);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (EPI == EPI_F32) {
        if (args.splits > 1 || args.beta != 0.f)
          tma_reduce_add_2d(maps.C, slot, col0, row0);
        else
          tma_store_2d(maps.C, slot, col0, row0);
      } else if (EPI == EPI_BIAS_GELU) {
        tma_store_2d(maps.aux, slot, col0, row0);
        tma_store_2d(maps.C, slot + kEpiSlot, col0, row0);
      } else {
#if ZB_GEMM_EXP != 1  // experiment 1: no output stores
        tma_store_2d(maps.C, slot, col0, row0);
#endif
      }
      bulk_commit();
    }
    if (BIAS) {
#pragma unroll
      for (int j = 0; j < 4; ++j) bq[j] = bn[j];
    }
  }
}

template <int BN, int A_MN, int B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmC,
                      const __grid_constant__ CUtensorMap tmAux,
                      const __grid_constant__ CUtensorMap tmR, GemmArgs args) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B atoms.
  uint32_t base = smem_u32(smem_raw);
  uint32_t pad = ((base + 1023u) & ~1023u) - base;
  uint8_t* smem = smem_raw + pad;
  uint8_t* smA = smem;
  uint8_t* smB = smem + S * Cfg::A_BYTES;
  uint8_t* smE = smem + S * Cfg::STAGE_BYTES;  // epilogue staging, 4 KB per warp
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smE + Cfg::EPI_BYTES);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* epi_bar = tempty_bar + 2;  // [8 warps][2 slots]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_bar + 2 * kEpiWarps);

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
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&epi_bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // prologue above overlapped the previous kernel's tail (PDL launch)
  griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        int mt, nt;
        tile_mn(args, tile, mt, nt);
        const int m0 = mt * BM;
        const int n0 = nt * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
#if ZB_GEMM_EXP == 3  // experiment: no operand loads (time without TMA traffic)
          mbar_arrive(&full_bar[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          continue;
#endif
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
#if ZB_GEMM_EXP != 2  // experiment 2: no MMAs (time without tensor work)
            mma_bf16_ss(d_tmem, a_desc, b_desc, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
#endif
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
    const int part = (warp - 4) >> 2;  // which run of the tile's column chunks it drains
    const int cb = epi_cb(part, BN / 32), ce = epi_cb(part + 1, BN / 32);
    int local = 0;
    if (args.tma_epi) {
      const EpiMaps maps{&tmC, &tmAux, &tmR};
      uint8_t* stg = smE + (warp - 4) * Cfg::NS * kEpiSlot;
      uint64_t* ebar = epi_bar + 2 * (warp - 4);
      uint32_t eph = 0, ecnt = 0;
      for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
        const int tile = unit % num_tiles;
        const int acc = local & 1;
        int mt, nt;
        tile_mn(args, tile, mt, nt);
        const int m0 = mt * BM;
        const int n0 = nt * BN;
        epilogue_tma<EPI, Cfg::NS>(args, maps, stg, ebar, eph, ecnt,
                          tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN, &tfull_bar[acc],
                          (local >> 1) & 1, m0 + ew * 32, n0, cb, ce, lane,
                          [&] { if (lane == 0) mbar_arrive(&tempty_bar[acc]); });
      }
      if (lane == 0) bulk_wait_all();
    } else
    for (int unit = blockIdx.x; unit < num_units; unit += gridDim.x, ++local) {
      const int tile = unit % num_tiles;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      int mt, nt;
      tile_mn(args, tile, mt, nt);
      const int m0 = mt * BM;
      const int n0 = nt * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const bool row_ok = row < args.M;
#pragma unroll 1
      for (int c = cb; c < ce; ++c) {
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
  static constexpr int NS = epi_slots(STAGE_BYTES);
  static constexpr int EPI_BYTES = kEpiWarps * NS * 2048;
  static constexpr int FIT = (kSmemMax - 1536 - EPI_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = FIT < 8 ? FIT : 8;
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 512;
};

// MC = CTA pairs per cluster (cluster dims 2 * MC, set at launch).  MC = 2: the two pairs
// compute the two adjacent n-tiles of one m-tile and share its A operand: each CTA loads
// half of its 128 A rows and multicasts it to the same-rank CTA of the other pair, so A
// crosses L2 -> SM once per cluster (25% less operand traffic per SM at BN = 256).  A
// stage is refilled only after both pairs' MMAs released it (empty barrier count MC,
// commits multicast to the whole cluster).
template <int BN, int A_MN, int B_MN, int EPI, int MC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm2cta_kernel(const __grid_constant__ CUtensorMap tmA,
                    const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC,
                    const __grid_constant__ CUtensorMap tmAux,
                    const __grid_constant__ CUtensorMap tmR, GemmArgs args) {
  using Cfg = Gemm2Cfg<BN>;
  constexpr int S = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint32_t base = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base + 1023u) & ~1023u) - base);
  uint8_t* smA = smem;
  uint8_t* smB = smem + S * Cfg::A_BYTES;
  uint8_t* smE = smem + S * Cfg::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smE + Cfg::EPI_BYTES);
  uint64_t* empty_bar = full_bar + S;
  uint64_t* tfull_bar = empty_bar + S;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* epi_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_bar + 2 * kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;        // rank within the CTA pair
  const int pr = (int)(crank >> 1);      // pair within the cluster (MC = 2)
  const bool leader = rank == 0;
  const uint32_t lead_rank = crank & ~1u;  // this pair's leader in the cluster
  const int nv = args.num_n_tiles / MC;  // n-tile groups (one n-tile per pair)
  const int num_tiles = args.num_m_tiles * nv;  // m tiles of 256 rows x n-tile groups
  const int num_units = num_tiles * args.splits;
  const int num_kb = (args.K + BK - 1) / BK;
  const int cluster = blockIdx.x / (2 * MC), nclusters = gridDim.x / (2 * MC);
  auto coords = [&](int tile, int& mt, int& nt) {
    int g;
    if (args.n_fastest) {
      g = tile % nv;
      mt = tile / nv;
    } else {
      mt = tile % args.num_m_tiles;
      g = tile / args.num_m_tiles;
    }
    nt = g * MC + pr;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);   // leader's expect_tx (both CTAs' TMA bytes land here)
      mbar_init(&empty_bar[i], MC);  // one multicast MMA commit per pair
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], 2 * kEpiWarps);  // both CTAs' epilogue warps (leader's copy)
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&epi_bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_2cta(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // prologue above overlapped the previous kernel's tail (PDL launch)
  griddep_launch();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int unit = cluster; unit < num_units; unit += nclusters) {
        const int tile = unit % num_tiles;
        const int kb0 = (unit / num_tiles) * args.kb_per_split;
        const int kb1 = min(num_kb, kb0 + args.kb_per_split);
        int mt, nt;
        coords(tile, mt, nt);
        const int m0 = mt * 256 + (int)rank * 128;
        const int n0 = nt * BN + (int)rank * (BN / 2);
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
          if (MC == 2) {  // this CTA's half of the shared A rows, to both pairs
            const uint16_t mask = (uint16_t)((1u << rank) | (1u << (2 + rank)));
            if (A_MN)
              tma_load_2d_2cta_mc(a_dst + pr * (64 * BK * 2), &tmA, &full_bar[stage],
                                  m0 + pr * 64, k0, mask);
            else
              tma_load_2d_2cta_mc(a_dst + pr * (64 * 128), &tmA, &full_bar[stage], k0,
                                  m0 + pr * 64, mask);
          } else if (A_MN) {
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
          mma_commit_2cta_mask(&empty_bar[stage], (uint16_t)((1u << (2 * MC)) - 1));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_2cta_mask(&tfull_bar[acc], (uint16_t)(3u << lead_rank));
      }
    }
  } else if (warp >= 4) {
    const int ew = (warp - 4) & 3;
    const int part = (warp - 4) >> 2;
    const int cb = epi_cb(part, BN / 32), ce = epi_cb(part + 1, BN / 32);
    int local = 0;
    if (args.tma_epi) {
      const EpiMaps maps{&tmC, &tmAux, &tmR};
      uint8_t* stg = smE + (warp - 4) * Cfg::NS * kEpiSlot;
      uint64_t* ebar = epi_bar + 2 * (warp - 4);
      uint32_t eph = 0, ecnt = 0;
      for (int unit = cluster; unit < num_units; unit += nclusters, ++local) {
        const int tile = unit % num_tiles;
        const int acc = local & 1;
        int mt, nt;
        coords(tile, mt, nt);
        const int m0 = mt * 256 + (int)rank * 128;
        const int n0 = nt * BN;
        epilogue_tma<EPI, Cfg::NS>(args, maps, stg, ebar, eph, ecnt,
                          tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN, &tfull_bar[acc],
                          (local >> 1) & 1, m0 + ew * 32, n0, cb, ce, lane, [&] {
                            if (lane == 0) {
                              if (leader)
                                mbar_arrive(&tempty_bar[acc]);
                              else
                                mbar_arrive_remote(&tempty_bar[acc], lead_rank);
                            }
                          });
      }
      if (lane == 0) bulk_wait_all();
    } else
    for (int unit = cluster; unit < num_units; unit += nclusters, ++local) {
      const int tile = unit % num_tiles;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      int mt, nt;
      coords(tile, mt, nt);
      const int m0 = mt * 256 + (int)rank * 128;
      const int n0 = nt * BN;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      const bool row_ok = row < args.M;
#pragma unroll 1
      for (int c = cb; c < ce; ++c) {
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
          mbar_arrive_remote(&tempty_bar[acc], lead_rank);
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

struct EpiTm {
  CUtensorMap c, aux, r;
};

// Epilogue tile map: {32 columns, 32 rows} box; bf16 rows of 64 B use the 64-byte
// swizzle, fp32 rows of 128 B the 128-byte swizzle (see sw64 / sw128).
static int make_tmap_epi(CUtensorMap* m, const void* ptr, bool f32, uint64_t cols, uint64_t rows,
                         uint64_t ld) {
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * (f32 ? 4 : 2)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return tensor_map_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Launch with programmatic stream serialisation (PDL): the GEMM's prologue overlaps
// the previous kernel's tail; the kernel waits (griddep_wait) before any global access.
template <typename Kern, typename... Args>
static cudaError_t launch_pdl(Kern kern, dim3 grid, int smem, cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Same with a thread-block-cluster dimension (the 2-CTA kernels: 2 or 4 CTAs).
template <typename Kern, typename... Args>
static cudaError_t launch_pdl_cluster(Kern kern, dim3 grid, int smem, cudaStream_t stream,
                                      int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster_x;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <int BN, int A_MN, int B_MN, int EPI>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const EpiTm& et,
                       GemmArgs args, cudaStream_t stream) {
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
  const int splits = (EPI == EPI_F32 && args.beta == 1.f) ? (args.splits > 0 ? args.splits : 1) : 1;
  args.kb_per_split = (num_kb + splits - 1) / splits;
  args.splits = (num_kb + args.kb_per_split - 1) / args.kb_per_split;
  const int units = tiles * args.splits;
  int grid = units < num_sms() ? units : num_sms();
  cudaError_t e = launch_pdl(kern, dim3(grid), Cfg::SMEM_BYTES, stream, ta, tb, et.c, et.aux, et.r,
                             args);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  return 0;
}

// Co-resident 2-CTA clusters for a kernel with `smem` bytes of dynamic shared memory.
static int max_active_pairs(const void* kern, int smem, int csize = 2) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(csize * (num_sms() / csize));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = num_sms() / csize;
  }
  return n < num_sms() / csize ? n : num_sms() / csize;
}

// Slots for the tile cost model (all 2-CTA configurations use ~225 KB of smem).
static int pair_slots() {
  static int n = 0;
  if (!n) {
    auto k = gemm2cta_kernel<256, 0, 0, EPI_BF16, 1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Gemm2Cfg<256>::SMEM_BYTES);
    n = max_active_pairs((const void*)k, Gemm2Cfg<256>::SMEM_BYTES);
  }
  return n;
}

template <int BN, int A_MN, int B_MN, int EPI, int MC>
static int launch_gemm2(const CUtensorMap& ta, const CUtensorMap& tb, const EpiTm& et,
                        GemmArgs args, cudaStream_t stream) {
  using Cfg = Gemm2Cfg<BN>;
  auto kern = gemm2cta_kernel<BN, A_MN, B_MN, EPI, MC>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm2cta: cudaFuncSetAttribute");
    configured = true;
  }
  args.num_m_tiles = (args.M + 255) / 256;
  args.num_n_tiles = (args.N + BN - 1) / BN;
  if (args.num_n_tiles % MC)
    return set_error(ZB_ERR_INVALID, "gemm: multicast pairs need an even n-tile count");
  const int tiles = args.num_m_tiles * (args.num_n_tiles / MC);
  const int num_kb = (args.K + BK - 1) / BK;
  // A persistent grid must be fully co-resident: not every SM pair can host a
  // cluster (GPC shapes), so ask the occupancy API instead of assuming sms / 2.
  static int max_clusters = 0;
  if (!max_clusters)
    max_clusters = max_active_pairs((const void*)kern, Cfg::SMEM_BYTES, 2 * MC);
  const int pairs = max_clusters;
  const int splits = (EPI == EPI_F32 && args.beta == 1.f) ? (args.splits > 0 ? args.splits : 1) : 1;
  args.kb_per_split = (num_kb + splits - 1) / splits;
  args.splits = (num_kb + args.kb_per_split - 1) / args.kb_per_split;
  const int units = tiles * args.splits;
  const int clusters = units < pairs ? units : pairs;
  cudaError_t e = launch_pdl_cluster(kern, dim3(2 * MC * clusters), Cfg::SMEM_BYTES, stream,
                                     2 * MC, ta, tb, et.c, et.aux, et.r, args);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, "gemm2cta launch");
  return 0;
}

template <int BN, int A_MN, int B_MN, int MC = 1>
static int dispatch_epi2(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const EpiTm& et,
                         GemmArgs args, cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch_gemm2<BN, A_MN, B_MN, EPI_BF16, MC>(ta, tb, et, args, s);
    case EPI_BIAS: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS, MC>(ta, tb, et, args, s);
    case EPI_BIAS_GELU: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS_GELU, MC>(ta, tb, et, args, s);
    case EPI_BIAS_RESID: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS_RESID, MC>(ta, tb, et, args, s);
    case EPI_GELU_BWD: return launch_gemm2<BN, A_MN, B_MN, EPI_GELU_BWD, MC>(ta, tb, et, args, s);
    case EPI_F32: return launch_gemm2<BN, A_MN, B_MN, EPI_F32, MC>(ta, tb, et, args, s);
    case EPI_RESID: return launch_gemm2<BN, A_MN, B_MN, EPI_RESID, MC>(ta, tb, et, args, s);
    case EPI_BIAS_GELU_NA: return launch_gemm2<BN, A_MN, B_MN, EPI_BIAS_GELU_NA, MC>(ta, tb, et, args, s);
  }
  return set_error(ZB_ERR_INVALID, "gemm: unknown epilogue %d", epi);
}

template <int BN, int A_MN, int B_MN>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, const EpiTm& et,
                         GemmArgs args, cudaStream_t s) {
  switch (epi) {
    case EPI_BF16: return launch_gemm<BN, A_MN, B_MN, EPI_BF16>(ta, tb, et, args, s);
    case EPI_BIAS: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS>(ta, tb, et, args, s);
    case EPI_BIAS_GELU: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS_GELU>(ta, tb, et, args, s);
    case EPI_BIAS_RESID: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS_RESID>(ta, tb, et, args, s);
    case EPI_GELU_BWD: return launch_gemm<BN, A_MN, B_MN, EPI_GELU_BWD>(ta, tb, et, args, s);
    case EPI_F32: return launch_gemm<BN, A_MN, B_MN, EPI_F32>(ta, tb, et, args, s);
    case EPI_RESID: return launch_gemm<BN, A_MN, B_MN, EPI_RESID>(ta, tb, et, args, s);
    case EPI_BIAS_GELU_NA: return launch_gemm<BN, A_MN, B_MN, EPI_BIAS_GELU_NA>(ta, tb, et, args, s);
  }
  return set_error(ZB_ERR_INVALID, "gemm: unknown epilogue %d", epi);
}

// ---------------------------------------------------------------- tile selection
struct GemmChoice {
  int pair, bn, splits;
};

// Wave-quantisation cost model (SM cycles), calibrated on B200 (scripts/gemm_sweep.py,
// profiles/r01_gemm_sweep.jsonl): per k-block a 128 x BN tile costs 512 / 400 / 360
// cycles for BN = 256 / 192 / 128 (smaller tiles are operand-bandwidth bound), a
// 256 x BN CTA-pair tile 480 / 380 per SM; each (tile, K-split) unit adds fill /
// drain; fp32 accumulation (beta = 1) may split K and pays the TMA reduce-add of
// every split's partial tile at ~1500 B/cycle of L2 reduction bandwidth.
static GemmChoice model_choice(int M, int N, int K, int a_mn, int b_mn, int epilogue, float beta,
                               int force) {
  GemmChoice best_c{0, 256, 1};
  const bool pair_ok = force == 2 || (kPairTilesDefault && force != 1 && M >= 256 &&
                                      !(b_mn && !a_mn));
  const int sms = num_sms();
  const int nkb = (K + BK - 1) / BK;
  const bool can_split = epilogue == EPI_F32 && beta == 1.f;
  const int max_s = can_split ? (nkb / 4 < 16 ? (nkb / 4 > 1 ? nkb / 4 : 1) : 16) : 1;
  double best = 1e30;
  for (int two = 0; two <= 1; ++two) {
    if (two && (!pair_ok || M < 256)) continue;
    if (!two && force == 2 && M >= 256) continue;
    for (int bn : {256, 192, 128}) {
      if (two && bn == 128) continue;
      if (two && b_mn && bn == 192) continue;  // MN-major half-tiles must be 64-multiples
      const long long t = (long long)((M + (two ? 255 : 127)) / (two ? 256 : 128)) * ((N + bn - 1) / bn);
      const long long slots = two ? pair_slots() : sms;
      const double per = two ? (bn == 256 ? 480.0 : 380.0)
                             : (bn == 256 ? 512.0 : (bn == 192 ? 400.0 : 360.0));
      const double fixed = two ? 2000.0 : 800.0;
      for (int sp = 1; sp <= max_s; ++sp) {
        const long long units = t * sp;
        const long long waves = (units + slots - 1) / slots;
        const int kbs = (nkb + sp - 1) / sp;
        double cost = waves * (kbs * per + fixed);
        if (can_split) cost += (double)sp * M * N * 4.0 / 1500.0;
        if (cost < best - 1e-9) {
          best = cost;
          best_c = {two, bn, sp};
        }
      }
    }
  }
  if (N <= 128 && !best_c.pair) best_c.bn = 128;
  return best_c;
}

struct GemmKey {
  int M, N, K, a_mn, b_mn, epi, beta1, ldc;
  bool operator<(const GemmKey& o) const {
    return std::tie(M, N, K, a_mn, b_mn, epi, beta1, ldc) <
           std::tie(o.M, o.N, o.K, o.a_mn, o.b_mn, o.epi, o.beta1, o.ldc);
  }
};
static std::mutex g_tune_mu;
static std::map<GemmKey, GemmChoice> g_tuned;

// Tile table measured on B200 (scripts/tune_gemm.py): gemm_tune_cache.txt beside this
// library, one line per shape "g1 M N K a_mn b_mn epi beta1 ldc pair bn splits".  The
// library only READS it (once, on the first call); entries whose tag is not the
// current kernel generation kTileTableTag are ignored, so tilings measured on older
// kernels never outlive a kernel change.  Shapes not in the table use the cost model.
static const char* kTileTableTag = "g1";

static std::string tune_cache_path() {
  Dl_info info;
  if (dladdr((void*)&tune_cache_path, &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t k = so.find_last_of('/');
    return (k == std::string::npos ? std::string(".") : so.substr(0, k)) + "/gemm_tune_cache.txt";
  }
  return "gemm_tune_cache.txt";
}

static void tune_cache_load() {
  static bool loaded = false;
  if (loaded) return;
  loaded = true;
  FILE* f = fopen(tune_cache_path().c_str(), "r");
  if (!f) return;
  char line[256], tag[16];
  while (fgets(line, sizeof(line), f)) {
    GemmKey k;
    GemmChoice c;
    if (sscanf(line, "%15s %d %d %d %d %d %d %d %d %d %d %d", tag, &k.M, &k.N, &k.K, &k.a_mn,
               &k.b_mn, &k.epi, &k.beta1, &k.ldc, &c.pair, &c.bn, &c.splits) != 12)
      continue;
    if (strcmp(tag, kTileTableTag) != 0) continue;
    if ((c.bn == 128 || c.bn == 192 || c.bn == 256) && c.splits >= 1 && (c.pair >= 0 && c.pair <= 2))
      g_tuned[k] = c;
  }
  fclose(f);
}

struct GemmCall {
  const void *A, *B, *bias, *R;
  int M, N, K, lda, ldb, ldc, ldr, ldaux, a_mn, b_mn, epilogue;
  float beta;
};

// raster: -1 = by operand size, 0 = M-fastest, 1 = N-fastest; allow_tma_epi: 0 forces
// the direct-store epilogue (tests / experiments only).
static int launch_choice(const GemmCall& g, const GemmChoice& ch, void* C, void* aux,
                         cudaStream_t stream, int raster = -1, int allow_tma_epi = 1) {
  const int BN = ch.bn, pair = ch.pair;
  CUtensorMap ta, tb;
  int rc;
  if (g.a_mn)
    rc = make_tmap(&ta, g.A, (uint64_t)g.M, (uint64_t)g.K, (uint64_t)g.lda, BK);
  else
    rc = make_tmap(&ta, g.A, (uint64_t)g.K, (uint64_t)g.M, (uint64_t)g.lda,
                   pair == 2 ? BM / 2 : BM);  // multicast pairs: half the rows per CTA
  if (rc) return rc;
  if (g.b_mn)
    rc = make_tmap(&tb, g.B, (uint64_t)g.N, (uint64_t)g.K, (uint64_t)g.ldb, BK);
  else
    rc = make_tmap(&tb, g.B, (uint64_t)g.K, (uint64_t)g.N, (uint64_t)g.ldb,
                   (uint32_t)(pair ? BN / 2 : BN));
  if (rc) return rc;
  GemmArgs args{};
  args.C = C;
  args.bias = reinterpret_cast<const __nv_bfloat16*>(g.bias);
  args.R = reinterpret_cast<const __nv_bfloat16*>(g.R);
  args.aux = reinterpret_cast<__nv_bfloat16*>(aux);
  args.M = g.M; args.N = g.N; args.K = g.K;
  args.ldc = g.ldc; args.ldr = g.ldr; args.ldaux = g.ldaux;
  args.beta = g.beta;
  args.splits = ch.splits;
  {
    const uint64_t a_bytes = (uint64_t)g.M * g.K * 2, b_bytes = (uint64_t)g.N * g.K * 2;
    args.n_fastest = raster >= 0 ? raster : (a_bytes > b_bytes && a_bytes > (64ull << 20));
  }
  const int epilogue = g.epilogue;
  {
    const int celem = (epilogue == EPI_F32) ? 4 : 8;  // elements per 16 bytes
    bool v = (g.ldc % celem) == 0 && ((uintptr_t)C & 15) == 0;
    if (g.R) v = v && (g.ldr % 8) == 0 && ((uintptr_t)g.R & 15) == 0;
    if (aux) v = v && (g.ldaux % 8) == 0 && ((uintptr_t)aux & 15) == 0;
    if (g.bias) v = v && ((uintptr_t)g.bias & 15) == 0;
    args.vec = v ? 1 : 0;
  }
  // TMA-store epilogue: C / aux / R tile maps with a {32 cols, 32 rows} box (64-byte
  // swizzle for bf16 rows, 128-byte for fp32).  Needs 16-byte aligned bases and
  // pitches, and fp32 accumulation only as beta in {0, 1} (TMA reduce-add).
  EpiTm et;
  std::memset(&et, 0, sizeof(et));
  {
    const bool f32 = epilogue == EPI_F32;
    const int esz = f32 ? 4 : 2;
    bool ok = ((uintptr_t)C & 15) == 0 && ((size_t)g.ldc * esz) % 16 == 0;
    if (f32) ok = ok && (g.beta == 0.f || g.beta == 1.f);
    if (aux) ok = ok && ((uintptr_t)aux & 15) == 0 && (g.ldaux % 8) == 0;
    if (g.R) ok = ok && ((uintptr_t)g.R & 15) == 0 && (g.ldr % 8) == 0;
    if (epilogue == EPI_BIAS_GELU || epilogue == EPI_GELU_BWD) ok = ok && aux;
    if (epilogue == EPI_BIAS_RESID || epilogue == EPI_RESID) ok = ok && g.R;
    if (!allow_tma_epi) ok = false;
    if (ok) {
      int rc2 = make_tmap_epi(&et.c, C, f32, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldc);
      if (!rc2 && aux)
        rc2 = make_tmap_epi(&et.aux, aux, false, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldaux);
      if (!rc2 && g.R)
        rc2 = make_tmap_epi(&et.r, g.R, false, (uint64_t)g.N, (uint64_t)g.M, (uint64_t)g.ldr);
      if (rc2) return rc2;
    }
    args.tma_epi = ok ? 1 : 0;
  }
  const int key = g.a_mn * 2 + g.b_mn;
  if (pair == 2) {
    if (BN == 256) {
      switch (key) {
        case 0: return dispatch_epi2<256, 0, 0, 2>(epilogue, ta, tb, et, args, stream);
        case 1: return dispatch_epi2<256, 0, 1, 2>(epilogue, ta, tb, et, args, stream);
        case 3: return dispatch_epi2<256, 1, 1, 2>(epilogue, ta, tb, et, args, stream);
      }
    } else if (BN == 192) {
      switch (key) {
        case 0: return dispatch_epi2<192, 0, 0, 2>(epilogue, ta, tb, et, args, stream);
      }
    }
    return set_error(ZB_ERR_INVALID, "gemm: unsupported multicast-pair layout");
  }
  if (pair) {
    if (BN == 256) {
      switch (key) {
        case 0: return dispatch_epi2<256, 0, 0>(epilogue, ta, tb, et, args, stream);
        case 1: return dispatch_epi2<256, 0, 1>(epilogue, ta, tb, et, args, stream);
        case 3: return dispatch_epi2<256, 1, 1>(epilogue, ta, tb, et, args, stream);
      }
    } else if (BN == 192) {
      switch (key) {
        case 0: return dispatch_epi2<192, 0, 0>(epilogue, ta, tb, et, args, stream);
      }
    } else {
      switch (key) {
        case 0: return dispatch_epi2<128, 0, 0>(epilogue, ta, tb, et, args, stream);
        case 1: return dispatch_epi2<128, 0, 1>(epilogue, ta, tb, et, args, stream);
        case 3: return dispatch_epi2<128, 1, 1>(epilogue, ta, tb, et, args, stream);
      }
    }
    return set_error(ZB_ERR_INVALID, "gemm: unsupported 2-CTA layout");
  }
  if (BN == 256) {
    switch (key) {
      case 0: return dispatch_epi<256, 0, 0>(epilogue, ta, tb, et, args, stream);
      case 1: return dispatch_epi<256, 0, 1>(epilogue, ta, tb, et, args, stream);
      case 3: return dispatch_epi<256, 1, 1>(epilogue, ta, tb, et, args, stream);
    }
  } else if (BN == 192) {
    switch (key) {
      case 0: return dispatch_epi<192, 0, 0>(epilogue, ta, tb, et, args, stream);
      case 1: return dispatch_epi<192, 0, 1>(epilogue, ta, tb, et, args, stream);
      case 3: return dispatch_epi<192, 1, 1>(epilogue, ta, tb, et, args, stream);
    }
  } else {
    switch (key) {
      case 0: return dispatch_epi<128, 0, 0>(epilogue, ta, tb, et, args, stream);
      case 1: return dispatch_epi<128, 0, 1>(epilogue, ta, tb, et, args, stream);
      case 3: return dispatch_epi<128, 1, 1>(epilogue, ta, tb, et, args, stream);
    }
  }
  return set_error(ZB_ERR_INVALID, "gemm: unsupported layout (A MN-major with B K-major)");
}

// Measured choice (zb_gemm_tune, called by scripts/tune_gemm.py only): time the
// model's pick and its neighbours on scratch outputs (inputs are only read), keep
// the fastest.  Synchronises the stream; never called by zb_gemm_bf16.
static GemmChoice tune_choice(const GemmCall& g, const GemmChoice& model, void* aux_ro,
                              cudaStream_t stream) {
  std::vector<GemmChoice> cands{model};
  const bool can_split = g.epilogue == EPI_F32 && g.beta == 1.f;
  const int nkb = (g.K + BK - 1) / BK;
  for (int bn : {256, 192, 128})
    for (int sp : {1, 2, 4, 8}) {
      if (sp > 1 && (!can_split || nkb / sp < 4)) continue;
      cands.push_back({0, bn, sp});
      if (g.M >= 256 && bn != 128 && !(g.b_mn && !g.a_mn) && !(g.b_mn && bn == 192))
        cands.push_back({1, bn, sp});
      // multicast pairs: two CTA pairs share the A tile (even n-tile count)
      if (g.M >= 256 && bn != 128 && !(g.b_mn && bn == 192) && ((g.N + bn - 1) / bn) % 2 == 0)
        cands.push_back({2, bn, sp});
    }
  const size_t esz = g.epilogue == EPI_F32 ? 4 : 2;
  void *c = nullptr, *x = nullptr;
  // stream-ordered scratch (no device-wide synchronisation while other streams,
  // e.g. peer collectives, are in flight)
  if (cudaMallocAsync(&c, (size_t)g.ldc * g.M * esz, stream) != cudaSuccess) {
    cudaGetLastError();
    return model;
  }
  if (g.epilogue == EPI_BIAS_GELU &&
      cudaMallocAsync(&x, (size_t)g.ldaux * g.M * 2, stream) != cudaSuccess) {
    cudaGetLastError();
    cudaFreeAsync(c, stream);
    return model;
  }
  void* aux = g.epilogue == EPI_BIAS_GELU ? x : nullptr;
  if (g.epilogue == EPI_GELU_BWD) aux = aux_ro;  // read-only operand
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  GemmChoice best = model;
  float best_ms = 1e30f;
  for (const GemmChoice& ch : cands) {
    bool ok = true;
    for (int w = 0; w < 2 && ok; ++w) ok = launch_choice(g, ch, c, aux, stream) == 0;
    if (!ok) continue;
    cudaEventRecord(e0, stream);
    for (int it = 0; it < 5 && ok; ++it) ok = launch_choice(g, ch, c, aux, stream) == 0;
    cudaEventRecord(e1, stream);
    if (!ok || cudaEventSynchronize(e1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_ms * 0.98f) {  // keep the model's pick unless clearly beaten
      best_ms = ms;
      best = ch;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFreeAsync(c, stream);
  if (x) cudaFreeAsync(x, stream);
  return best;
}

static int gemm_validate(const void* A, const void* B, const void* bias, const void* R,
                         const void* aux, int M, int N, int K, int lda, int ldb, int epilogue) {
  if (M <= 0 || N <= 0 || K <= 0) return set_error(ZB_ERR_INVALID, "gemm: bad shape %d %d %d", M, N, K);
  if ((lda % 8) || (ldb % 8))
    return set_error(ZB_ERR_INVALID, "gemm: lda/ldb must be multiples of 8 elements");
  if (((uintptr_t)A & 15) || ((uintptr_t)B & 15))
    return set_error(ZB_ERR_INVALID, "gemm: A/B must be 16-byte aligned");
  if (epilogue < EPI_BF16 || epilogue > EPI_BIAS_GELU_NA)
    return set_error(ZB_ERR_INVALID, "gemm: unknown epilogue %d", epilogue);
  const bool needs_bias = epilogue == EPI_BIAS || epilogue == EPI_BIAS_GELU ||
                          epilogue == EPI_BIAS_RESID || epilogue == EPI_BIAS_GELU_NA;
  if (needs_bias && !bias) return set_error(ZB_ERR_INVALID, "gemm: epilogue %d needs bias", epilogue);
  if ((epilogue == EPI_BIAS_GELU || epilogue == EPI_GELU_BWD) && !aux)
    return set_error(ZB_ERR_INVALID, "gemm: epilogue %d needs aux", epilogue);
  if ((epilogue == EPI_BIAS_RESID || epilogue == EPI_RESID) && !R)
    return set_error(ZB_ERR_INVALID, "gemm: epilogue %d needs a residual", epilogue);
  return 0;
}

// The tile zb_gemm_bf16 uses: the measured table entry, else the cost model.
static GemmChoice default_choice(int M, int N, int K, int a_mn, int b_mn, int epilogue, float beta,
                                 int ldc, int* from_table) {
  const GemmKey key{M, N, K, a_mn, b_mn, epilogue, beta == 1.f ? 1 : 0, ldc};
  std::lock_guard<std::mutex> lk(g_tune_mu);
  tune_cache_load();
  auto it = g_tuned.find(key);
  if (from_table) *from_table = it != g_tuned.end();
  if (it != g_tuned.end()) return it->second;
  return model_choice(M, N, K, a_mn, b_mn, epilogue, beta, 0);
}

}  // namespace zb
using namespace zb;

extern "C" int zb_gemm_bf16(const void* A, const void* B, void* C, const void* bias,
                            const void* R, void* aux, int M, int N, int K, int lda, int ldb,
                            int ldc, int ldr, int ldaux, int a_mn_major, int b_mn_major,
                            int epilogue, float beta, cudaStream_t stream) {
  if (int rc = gemm_validate(A, B, bias, R, aux, M, N, K, lda, ldb, epilogue)) return rc;
  GemmCall g{A, B, bias, R, M, N, K, lda, ldb, ldc, ldr, ldaux, a_mn_major, b_mn_major,
             epilogue, beta};
  const GemmChoice ch = default_choice(M, N, K, a_mn_major, b_mn_major, epilogue, beta, ldc, nullptr);
  return launch_choice(g, ch, C, aux, stream);
}

extern "C" int zb_gemm_bf16_tile(const void* A, const void* B, void* C, const void* bias,
                                 const void* R, void* aux, int M, int N, int K, int lda, int ldb,
                                 int ldc, int ldr, int ldaux, int a_mn_major, int b_mn_major,
                                 int epilogue, float beta, int pair, int bn, int splits,
                                 int raster, int tma_epi, cudaStream_t stream) {
  if (int rc = gemm_validate(A, B, bias, R, aux, M, N, K, lda, ldb, epilogue)) return rc;
  GemmCall g{A, B, bias, R, M, N, K, lda, ldb, ldc, ldr, ldaux, a_mn_major, b_mn_major,
             epilogue, beta};
  GemmChoice ch = model_choice(M, N, K, a_mn_major, b_mn_major, epilogue, beta,
                               pair == 0 ? 1 : (pair > 0 ? 2 : 0));
  if (pair >= 0) ch.pair = pair;
  if (bn > 0) {
    if (bn != 128 && bn != 192 && bn != 256) return set_error(ZB_ERR_INVALID, "gemm: bn %d", bn);
    ch.bn = bn;
  }
  if (splits > 0) {
    if (splits > 1 && !(epilogue == EPI_F32 && beta == 1.f))
      return set_error(ZB_ERR_INVALID, "gemm: K splits need fp32 accumulation (beta = 1)");
    ch.splits = splits;
  }
  if (ch.pair && M < 256) return set_error(ZB_ERR_INVALID, "gemm: CTA-pair tiles need M >= 256");
  return launch_choice(g, ch, C, aux, stream, raster, tma_epi != 0);
}

extern "C" int zb_gemm_choice(int M, int N, int K, int a_mn_major, int b_mn_major, int epilogue,
                              float beta, int ldc, int* pair, int* bn, int* splits,
                              int* from_table) {
  if (!pair || !bn || !splits) return set_error(ZB_ERR_INVALID, "gemm_choice: NULL output");
  const GemmChoice ch = default_choice(M, N, K, a_mn_major, b_mn_major, epilogue, beta, ldc, from_table);
  *pair = ch.pair;
  *bn = ch.bn;
  *splits = ch.splits;
  return 0;
}

extern "C" int zb_gemm_tune(const void* A, const void* B, const void* bias, const void* R,
                            void* aux, int M, int N, int K, int lda, int ldb, int ldc, int ldr,
                            int ldaux, int a_mn_major, int b_mn_major, int epilogue, float beta,
                            int* pair, int* bn, int* splits, cudaStream_t stream) {
  if (int rc = gemm_validate(A, B, bias, R, aux, M, N, K, lda, ldb, epilogue)) return rc;
  if (!pair || !bn || !splits) return set_error(ZB_ERR_INVALID, "gemm_tune: NULL output");
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st != cudaStreamCaptureStatusNone)
    return set_error(ZB_ERR_INVALID, "gemm_tune: not allowed during graph capture");
  GemmCall g{A, B, bias, R, M, N, K, lda, ldb, ldc, ldr, ldaux, a_mn_major, b_mn_major,
             epilogue, beta};
  const GemmChoice model = model_choice(M, N, K, a_mn_major, b_mn_major, epilogue, beta, 0);
  const GemmChoice ch = tune_choice(g, model, aux, stream);
  *pair = ch.pair;
  *bn = ch.bn;
  *splits = ch.splits;
  return 0;
}
