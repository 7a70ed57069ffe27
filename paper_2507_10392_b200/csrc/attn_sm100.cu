// Causal flash attention on 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// Forward, one CTA per (128-query tile, head, sequence):
//   warp 0      TMA producer: Q once, then K/V tiles of 128 keys into a 2-stage ring
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T into a double-buffered TMEM
//               S tile, O += P_j V_j into a TMEM O accumulator (P from smem)
//   warp 2      TMEM allocator
//   warps 4..7  softmax: thread r owns query row r — reads its whole S row from
//               TMEM (no cross-thread reductions), online max/sum, writes the bf16
//               P row into a swizzled smem tile, rescales its O row in TMEM
//               (tcgen05.ld/st) only when its running max moved, then the
//               normalised O row + lse to global.
// The MMA warp issues S_{j+1} before waiting for P_j, so the tensor core computes
// the next scores while the softmax warps work.
//
// Layout as in attn.cu: qkv rows [q|k|v] (pitch ld), sequence b = rows [b*S, (b+1)*S).
#include "common.cuh"
#include "trace.cuh"
#include "zb_internal.h"

#include <cstdlib>
#include <type_traits>

namespace zb {
namespace fa {

constexpr int BQ = 128;   // queries per CTA (= TMEM lanes = softmax threads)
constexpr int BKV = 128;  // keys per block
constexpr int kThreads = 256;
constexpr float LOG2E = 1.4426950408889634f;

template <int D>
struct FwdSmem {
  // K/V ring depth: at D = 64 a block's MMAs take ~512 cycles, so 4 stages are
  // needed to keep the L2 -> smem latency off the critical path (208 KB).
  static constexpr int NST = (D == 64) ? 4 : 2;
  static constexpr int Q_BYTES = BQ * D * 2;
  static constexpr int K_BYTES = BKV * D * 2;
  static constexpr int V_BYTES = BKV * D * 2;
  static constexpr int P_BYTES = BQ * BKV * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + NST * K_BYTES;
  static constexpr int OFF_P = OFF_V + NST * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;  // barriers + alignment slack (<= 26 x 8 B)
};

// K-major SW128 descriptor for a [rows][64*nblk] tile stored as nblk 64-column
// blocks of rows*128 bytes each; kk = 16-element K step.
ZB_DEVICE uint64_t desc_kmajor(uint32_t base, int kk, int rows) {
  return umma_desc_sw128(base + (kk >> 2) * rows * 128 + (kk & 3) * 32, 16, 1024);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap tm_rows128,
               const __grid_constant__ CUtensorMap tm_rows64, __nv_bfloat16* __restrict__ out,
               float* __restrict__ lse, int S, int H, int n_seq, float scale) {
  // Persistent: each CTA walks (query tile, head, sequence) work items in
  // heavy-first order with a stride of gridDim.x; TMEM, barriers and the K/V /
  // S / P rings persist across items (ring positions are global block counters).
  using L = FwdSmem<D>;
  constexpr int NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;              // [NST]
  uint64_t* kv_empty = bar + 1 + NST;       // [NST]
  uint64_t* s_full = bar + 1 + 2 * NST;     // [2]
  uint64_t* s_empty = s_full + 2;           // [2]
  uint64_t* p_full = s_full + 4;            // [2]
  uint64_t* p_empty = s_full + 6;           // [2]
  // O-accumulation completions alternate between two barriers (PV block k commits
  // o_bar[k & 1]).  With one barrier, PV_k and PV_{k+1} could both complete before
  // the softmax warps poll for PV_k (the MMA may issue PV_{k+1} as soon as P_{k+1}
  // is handed over), and a parity wait cannot tell phase k from phase k+2.
  // Two barriers cannot run two phases ahead: P_{k+2} is handed over only after
  // PV_k was consumed.
  uint64_t* o_bar = s_full + 8;             // [2]
  uint64_t* q_empty = s_full + 10;          // all S MMAs of an item done -> Q reusable
  uint64_t* o_empty = s_full + 11;          // epilogue read O -> next item may overwrite
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = S / BQ;
  const int HD = H * D;
  const int per_q = H * n_seq;
  const int items = nqt * per_q;
  auto decode = [&](int t, int& qt, int& h, int& b) {
    qt = nqt - 1 - t / per_q;  // heavy (late) query tiles first
    const int rem = t % per_q;
    h = rem % H;
    b = rem / H;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_rows128);
    tma_prefetch_desc(&tm_rows64);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(o_empty, 4);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(&o_bar[0], 1);
    mbar_init(&o_bar[1], 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o = tmem + 256;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int g = 0, lt = 0;
      for (int t = blockIdx.x; t < items; t += gridDim.x, ++lt) {
        int qt, h, b;
        decode(t, qt, h, b);
        const int row0 = b * S;
        mbar_wait(q_empty, (lt & 1) ^ 1);
        mbar_arrive_expect_tx(q_full, L::Q_BYTES);
#pragma unroll
        for (int kc = 0; kc < D / 64; ++kc)
          tma_load_2d(sm + L::OFF_Q + kc * BQ * 128, &tm_rows128, q_full, h * D + kc * 64,
                      row0 + qt * BQ);
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g % NST;
          mbar_wait(&kv_empty[st], ((g / NST) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[st], L::K_BYTES + L::V_BYTES);
          uint8_t* kd = sm + L::OFF_K + st * L::K_BYTES;
          uint8_t* vd = sm + L::OFF_V + st * L::V_BYTES;
          const int kr = row0 + j * BKV;
#pragma unroll
          for (int kc = 0; kc < D / 64; ++kc)
            tma_load_2d(kd + kc * BKV * 128, &tm_rows128, &kv_full[st], HD + h * D + kc * 64, kr);
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
#pragma unroll
            for (int dc = 0; dc < D / 64; ++dc)
              tma_load_2d(vd + (kb * (D / 64) + dc) * 8192, &tm_rows64, &kv_full[st],
                          2 * HD + h * D + dc * 64, kr + kb * 64);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(BQ, BKV, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(BQ, D, 0, 1);
      const uint32_t q_base = smem_u32(sm + L::OFF_Q);
      int gbase = 0, lt = 0;
      for (int t = blockIdx.x; t < items; t += gridDim.x, ++lt) {
        int qt, h, b;
        decode(t, qt, h, b);
        const int nblk = qt + 1;
        auto issue_s = [&](int j) {
          const int gi = gbase + j;
          const int st = gi % NST, sb = gi & 1;
          mbar_wait(&kv_full[st], (gi / NST) & 1);
          mbar_wait(&s_empty[sb], ((gi >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm + L::OFF_K + st * L::K_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_bf16_ss(t_s[sb], desc_kmajor(q_base, kk, BQ), desc_kmajor(k_base, kk, BKV),
                        idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(&s_full[sb]);
          if (j == nblk - 1) mma_commit(q_empty);  // last read of this item's Q
        };
        mbar_wait(q_full, lt & 1);
        tc_fence_after();
        issue_s(0);
        for (int j = 0; j < nblk; ++j) {
          if (j + 1 < nblk) issue_s(j + 1);
          const int gi = gbase + j;
          const int st = gi % NST, sb = gi & 1;
          mbar_wait(&p_full[sb], (gi >> 1) & 1);
          if (j == 0) mbar_wait(o_empty, (lt & 1) ^ 1);  // previous item's O was read
          tc_fence_after();
          const uint32_t p_base = smem_u32(sm + L::OFF_P + sb * L::P_BYTES);
          const uint32_t v_base = smem_u32(sm + L::OFF_V + st * L::V_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t a = desc_kmajor(p_base, kk, BQ);
            const uint64_t bdesc =
                umma_desc_sw128(v_base + (kk >> 2) * (D / 64) * 8192 + (kk & 3) * 2048, 8192, 1024);
            mma_bf16_ss(t_o, a, bdesc, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&kv_empty[st]);
          mma_commit(&p_empty[sb]);
          mma_commit(&o_bar[gi & 1]);
        }
        gbase += nblk;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    const int wq = warp - 4;                 // TMEM lane quarter
    const int r = wq * 32 + lane;            // query row in the tile
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    // Running max in the scaled log2 domain.  It is only moved when a row's new
    // max exceeds it by more than RESCALE_T (P stays <= 2^RESCALE_T, exact in
    // fp32/bf16), so O is rarely rescaled and the softmax warps normally hand P_j
    // to the MMA warp without waiting for P_{j-1} V_{j-1}.
    constexpr float RESCALE_T = 8.f;
    int gbase = 0;
    int o_seen = 0;  // PV blocks known complete (global block counter)
    auto consume_o = [&](int upto) {
      while (o_seen < upto) {
        mbar_wait(&o_bar[o_seen & 1], (o_seen >> 1) & 1);
        ++o_seen;
      }
    };
    for (int t = blockIdx.x; t < items; t += gridDim.x) {
      int qt, h, b;
      decode(t, qt, h, b);
      const int nblk = qt + 1;
      const int q = qt * BQ + r;
      const int row0 = b * S;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nblk; ++j) {
        const int gi = gbase + j;
        const int sb = gi & 1;
        mbar_wait(&s_full[sb], (gi >> 1) & 1);
        tc_fence_after();
        // the whole S row in flight at once: one TMEM round trip instead of four
        float sv[BKV];
        uint32_t v[BKV / 32][32];
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c) tmem_ld_32x32b_x32(t_s[sb] + lane_off + c * 32, v[c]);
        tmem_ld_wait_regs(v[0]);
#pragma unroll
        for (int c = 1; c < BKV / 32; ++c) reg_tie(v[c]);
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(v[c][i]);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[sb]);
        if (j == qt) {  // diagonal block: keys after the query are masked
#pragma unroll
          for (int c = 0; c < BKV; ++c)
            if (c > r) sv[c] = -INFINITY;
        }
        // 8 independent max / sum chains (a single 128-long dependent chain costs
        // ~4 cycles per element of latency on one warp per scheduler)
        float mx8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mx8[i] = sv[i];
#pragma unroll
        for (int c = 8; c < BKV; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], sv[c]);
        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        mx *= sl2;
        const bool move = mx > m + RESCALE_T;
        const float m_new = move ? mx : m;
        const float corr = move ? exp2_fast(m - m_new) : 1.f;  // 0 on the first block
        m = m_new;
        float rs8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < BKV; ++c) {
          const float xe = fmaf(sv[c], sl2, -m);
          sv[c] = (c & 3) == 3 ? exp2_poly(xe) : exp2_fast(xe);  // 1/4 on the FMA pipe
          rs8[c & 7] += sv[c];
        }
        const float rs = ((rs8[0] + rs8[1]) + (rs8[2] + rs8[3])) + ((rs8[4] + rs8[5]) + (rs8[6] + rs8[7]));
        l = l * corr + rs;
        mbar_wait(&p_empty[sb], ((gi >> 1) & 1) ^ 1);
        uint8_t* prow = sm + L::OFF_P + sb * L::P_BYTES + r * 128;
#pragma unroll
        for (int ch = 0; ch < BKV / 8; ++ch) {
          uint4 pk;
          pk.x = pack_bf16(sv[ch * 8 + 0], sv[ch * 8 + 1]);
          pk.y = pack_bf16(sv[ch * 8 + 2], sv[ch * 8 + 3]);
          pk.z = pack_bf16(sv[ch * 8 + 4], sv[ch * 8 + 5]);
          pk.w = pack_bf16(sv[ch * 8 + 6], sv[ch * 8 + 7]);
          const int kb = ch >> 3, cc = ch & 7;
          *reinterpret_cast<uint4*>(prow + kb * (BQ * 128) + ((cc ^ (r & 7)) << 4)) = pk;
        }
        fence_proxy_async_smem();
        const bool rescale = j > 0 && __any_sync(0xffffffffu, move);
        if (rescale) {  // O must hold P_{j-1} V_{j-1} before it is rescaled
          consume_o(gi);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_o + lane_off + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(t_o + lane_off + c * 32, v);
          }
          tmem_st_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
        // keep o_bar consumption in step (PV_{gi-1} consumed before P_{gi+1} is handed over)
        consume_o(gi);
      }
      // epilogue: O / l -> bf16 row, lse
      consume_o(gbase + nblk);
      tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* orow = out + ((size_t)row0 + q) * HD + h * D;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_o + lane_off + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 pk;
          pk.x = pack_bf16(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          pk.y = pack_bf16(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
          pk.z = pack_bf16(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
          pk.w = pack_bf16(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + i) = pk;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
      lse[((size_t)b * H + h) * S + q] = (m + __log2f(l)) / LOG2E;
      gbase += nblk;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- D = 64: two CTAs per SM
// The single-CTA kernel above keeps each SM's tensor core idle while its one softmax
// warpgroup works (one warp per scheduler, nothing to hide its latencies).  Here P
// is written to TMEM (tcgen05.st) and the PV MMA reads it from there (A operand in
// TMEM), so a CTA needs only Q + a 2-stage K/V ring in smem (80 KB), 256 TMEM
// columns (S | P | O) and <= 128 registers per thread: two CTAs share every SM and
// one CTA's MMAs run while the other's softmax warps work.  The softmax makes two
// passes over the S row in TMEM (max, then exp / sum / pack) instead of holding
// 128 values in registers.
namespace fa_ts {
constexpr int BQ = 128, BKV = 128, D = 64, NST = 2, kThreads = 384;
constexpr int kSoft = 8;  // softmax warps: two per TMEM lane quarter, one per column half
constexpr float LOG2E = 1.4426950408889634f;
constexpr int Q_BYTES = BQ * D * 2, K_BYTES = BKV * D * 2, V_BYTES = BKV * D * 2;
constexpr int OFF_Q = 0, OFF_K = 2 * Q_BYTES, OFF_V = OFF_K + NST * K_BYTES;  // Q double-buffered
constexpr int OFF_X = OFF_V + NST * V_BYTES;  // [2 halves][128 rows] fp32 row-max / row-sum exchange
constexpr int OFF_BAR = OFF_X + 2 * BQ * 4;
constexpr int SMEM_BYTES = OFF_BAR + 256 + 1024;
constexpr uint32_t COL_S = 0, COL_P = 128, COL_O = 192, TMEM_COLS = 256;

__global__ void __launch_bounds__(kThreads, 2)
    fwd_ts_kernel(const __grid_constant__ CUtensorMap tm_rows128,
                  const __grid_constant__ CUtensorMap tm_rows64, __nv_bfloat16* __restrict__ out,
                  float* __restrict__ lse, int S, int H, int n_seq, float scale) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* q_full = bar + 0;     // [2] (the next item's Q loads during this item)
  uint64_t* q_empty = bar + 2;    // [2]
  uint64_t* kv_full = bar + 4;    // [NST]
  uint64_t* kv_empty = bar + 6;   // [NST]
  uint64_t* s_full = bar + 8;
  uint64_t* s_empty = bar + 9;    // softmax finished reading S
  uint64_t* p_full = bar + 10;    // P in TMEM (and any O rescale) done
  uint64_t* o_bar = bar + 11;     // [2] PV block k commits o_bar[k & 1] (see fwd_kernel)
  uint64_t* o_empty = bar + 13;   // epilogue read O
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 14);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqt = S / BQ;
  const int HD = H * D;
  const int per_q = H * n_seq;
  const int items = nqt * per_q;
  // Work items sorted heavy-first (late query tiles have the most key blocks), dealt
  // to the persistent CTAs in boustrophedon order (round k: CTA c takes rank
  // k*P + c for even k, k*P + P-1-c for odd k) so per-CTA totals even out.
  const int P = gridDim.x;
  auto item_of = [&](int k) { return k * P + ((k & 1) ? (P - 1 - (int)blockIdx.x) : (int)blockIdx.x); };
  auto decode = [&](int t, int& qt, int& h, int& b) {
    qt = nqt - 1 - t / per_q;  // heavy (late) query tiles first
    const int rem = t % per_q;
    h = rem % H;
    b = rem / H;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_rows128);
    tma_prefetch_desc(&tm_rows64);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, kSoft);
    mbar_init(p_full, kSoft);
    mbar_init(&o_bar[0], 1);
    mbar_init(&o_bar[1], 1);
    mbar_init(o_empty, kSoft);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t t_s = tmem + COL_S, t_p = tmem + COL_P, t_o = tmem + COL_O;
  griddep_wait();  // PDL: prologue overlapped the previous kernel's tail
  griddep_launch();

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int g = 0, lt = 0;
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int qt, h, b;
        decode(t, qt, h, b);
        const int row0 = b * S;
        const int qb = lt & 1;
        mbar_wait(&q_empty[qb], ((lt >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], Q_BYTES);
        tma_load_2d(sm + OFF_Q + qb * Q_BYTES, &tm_rows128, &q_full[qb], h * D, row0 + qt * BQ);
        for (int j = 0; j <= qt; ++j, ++g) {
          const int st = g % NST;
          mbar_wait(&kv_empty[st], ((g / NST) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[st], K_BYTES + V_BYTES);
          uint8_t* kd = sm + OFF_K + st * K_BYTES;
          uint8_t* vd = sm + OFF_V + st * V_BYTES;
          const int kr = row0 + j * BKV;
          tma_load_2d(kd, &tm_rows128, &kv_full[st], HD + h * D, kr);
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
            tma_load_2d(vd + kb * 8192, &tm_rows64, &kv_full[st], 2 * HD + h * D, kr + kb * 64);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(BQ, BKV, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(BQ, D, 0, 1);
      int gbase = 0, lt = 0;
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int qt, h, b;
        decode(t, qt, h, b);
        const int nblk = qt + 1;
        const int qb = lt & 1;
        const uint32_t q_base = smem_u32(sm + OFF_Q + qb * Q_BYTES);
        mbar_wait(&q_full[qb], (lt >> 1) & 1);
        for (int j = 0; j < nblk; ++j) {
          const int gi = gbase + j, st = gi % NST;
          mbar_wait(&kv_full[st], (gi / NST) & 1);
          mbar_wait(s_empty, (gi & 1) ^ 1);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm + OFF_K + st * K_BYTES);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_bf16_ss(t_s, desc_kmajor(q_base, kk, BQ), desc_kmajor(k_base, kk, BKV), idesc_s,
                        kk > 0 ? 1u : 0u);
          mma_commit(s_full);
          if (j == nblk - 1) mma_commit(&q_empty[qb]);
          mbar_wait(p_full, gi & 1);
          if (j == 0) mbar_wait(o_empty, (lt & 1) ^ 1);
          tc_fence_after();
          const uint32_t v_base = smem_u32(sm + OFF_V + st * V_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t bdesc =
                umma_desc_sw128(v_base + (kk >> 2) * 8192 + (kk & 3) * 2048, 8192, 1024);
            mma_bf16_ts(t_o, t_p + kk * 8, bdesc, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&kv_empty[st]);
          mma_commit(&o_bar[gi & 1]);
        }
        gbase += nblk;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue
    // Warp w owns rows of TMEM lane quarter (w-4)%4 and the column half (w-4)/4 of
    // every S / P / O tile; the two warps of a quarter exchange their partial row
    // maxima (and, at the end, row sums) through smem with a 64-thread named barrier.
    const int wq = (warp - 4) & 3, hf = (warp - 4) >> 2;
    const int r = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    float* xch = reinterpret_cast<float*>(sm + OFF_X);  // [2][BQ]
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + wq) : "memory"); };
    constexpr float RESCALE_T = 8.f;  // lazy O rescale (see fwd_kernel)
    int gbase = 0, o_seen = 0;
#ifdef ZB_EXP_TRACE
    long long acc_t[5] = {0, 0, 0, 0, 0}, t_start = clock64();
    int acc_n = 0;
#endif
    auto consume_o = [&](int upto) {
      while (o_seen < upto) {
        mbar_wait(&o_bar[o_seen & 1], (o_seen >> 1) & 1);
        ++o_seen;
      }
    };
    for (int k = 0, t = item_of(0); t < items; t = item_of(++k)) {
      int qt, h, b;
      decode(t, qt, h, b);
      const int nblk = qt + 1;
      const int q = qt * BQ + r;
      const int row0 = b * S;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nblk; ++j) {
        const int gi = gbase + j;
        const bool diag = j == qt;
#ifdef ZB_EXP_TRACE
        long long tr0 = clock64();
#endif
        mbar_wait(s_full, gi & 1);
        tc_fence_after();
#ifdef ZB_EXP_TRACE
        long long tr1 = clock64();
#endif
        // pass 1: max over this warp's 64 columns (masking only on the diagonal block)
        auto half_max = [&](auto diag_c) {
          constexpr bool DG = decltype(diag_c)::value;
          float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = hf * 2 + cc;
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_s + lane_off + c * 32, v);
            tmem_ld_wait_regs(v);
            float x[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              x[i] = __uint_as_float(v[i]);
              if (DG && c * 32 + i > r) x[i] = -INFINITY;
            }
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              mx4[0] = fmax3(mx4[0], x[i], x[i + 1]);
              mx4[1] = fmax3(mx4[1], x[i + 2], x[i + 3]);
              mx4[2] = fmax3(mx4[2], x[i + 4], x[i + 5]);
              mx4[3] = fmax3(mx4[3], x[i + 6], x[i + 7]);
            }
          }
          return fmaxf(fmax3(mx4[0], mx4[1], mx4[2]), mx4[3]);
        };
        const float mh = diag ? half_max(std::true_type{}) : half_max(std::false_type{});
        xch[hf * BQ + r] = mh;
        pair_sync();
        const float mx = fmaxf(mh, xch[(hf ^ 1) * BQ + r]) * sl2;
        pair_sync();  // both halves read before the next block overwrites
        const bool move = mx > m + RESCALE_T;
        const float m_new = move ? mx : m;
        const float corr = move ? exp2_fast(m - m_new) : 1.f;
        m = m_new;
#ifdef ZB_EXP_TRACE
        long long tr2 = clock64();
#endif
        // P (single TMEM buffer) and O are free once PV of the previous block is done
        consume_o(gi);
        tc_fence_after();
#ifdef ZB_EXP_TRACE
        long long tr3 = clock64();
#endif
        if (j > 0 && __any_sync(0xffffffffu, move)) {  // this half's 32 O columns
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_o + lane_off + hf * 32, v);
          tmem_ld_wait_regs(v);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
          tmem_st_32x32b_x32(t_o + lane_off + hf * 32, v);
        }
        // pass 2: exponentials, partial row sum, bf16 P into TMEM
        auto exp_pack = [&](auto diag_c) {
          constexpr bool DG = decltype(diag_c)::value;
          float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            const int c = hf * 2 + cc;
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_s + lane_off + c * 32, v);
            tmem_ld_wait_regs(v);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              // the SM's ex2 (MUFU) rate is the softmax floor: ~1/4 of the
              // exponentials go to the FMA pipe (exp2_poly)
              float p0 = exp2_fast(fmaf(__uint_as_float(v[i]), sl2, -m));
              const float x1 = fmaf(__uint_as_float(v[i + 1]), sl2, -m);
              float p1 = ((i >> 1) & 1) ? exp2_poly(x1) : exp2_fast(x1);
              if (DG && c * 32 + i > r) p0 = 0.f;
              if (DG && c * 32 + i + 1 > r) p1 = 0.f;
              rs4[(i >> 1) & 3] += p0 + p1;
              pk[i >> 1] = pack_bf16(p0, p1);
            }
            tmem_st_32x32b_x16(t_p + lane_off + c * 16, pk);
          }
          return (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
        };
        const float rs = diag ? exp_pack(std::true_type{}) : exp_pack(std::false_type{});
        l = l * corr + rs;  // this half's share of the row sum
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(s_empty);
          mbar_arrive(p_full);
        }
#ifdef ZB_EXP_TRACE
        long long tr4 = clock64();
        acc_t[0] += tr1 - tr0; acc_t[1] += tr2 - tr1; acc_t[2] += tr3 - tr2; acc_t[3] += tr4 - tr3;
        ++acc_n;
#endif
      }
      // epilogue: O / l -> bf16 row (this half's 32 columns), lse
      xch[hf * BQ + r] = l;
      pair_sync();
      const float lt = l + xch[(hf ^ 1) * BQ + r];
      pair_sync();
      consume_o(gbase + nblk);
      tc_fence_after();
      const float inv = 1.f / lt;
      __nv_bfloat16* orow = out + ((size_t)row0 + q) * HD + h * D + hf * 32;
      {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_o + lane_off + hf * 32, v);
        tmem_ld_wait_regs(v);
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 pk;
          pk.x = pack_bf16(__uint_as_float(v[i]) * inv, __uint_as_float(v[i + 1]) * inv);
          pk.y = pack_bf16(__uint_as_float(v[i + 2]) * inv, __uint_as_float(v[i + 3]) * inv);
          pk.z = pack_bf16(__uint_as_float(v[i + 4]) * inv, __uint_as_float(v[i + 5]) * inv);
          pk.w = pack_bf16(__uint_as_float(v[i + 6]) * inv, __uint_as_float(v[i + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + i) = pk;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(o_empty);
      if (hf == 0) lse[((size_t)b * H + h) * S + q] = (m + __log2f(lt)) / LOG2E;
      gbase += nblk;
    }
#ifdef ZB_EXP_TRACE  // per-CTA phase cycle totals (debug builds: build(defines=("ZB_EXP_TRACE",)))
    if (r == 0 && hf == 0 && (blockIdx.x == 0 || blockIdx.x == 100 || blockIdx.x == 250 || blockIdx.x == 295))
      printf("cta %d: blocks %d total %lld wait_s %lld pass1 %lld wait_o %lld pass2 %lld\n",
             blockIdx.x, acc_n, clock64() - t_start, acc_t[0], acc_t[1], acc_t[2], acc_t[3]);
#endif
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
}

static int run(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int ld, float scale,
               cudaStream_t s) {
  CUtensorMap m128, m64;
  const uint64_t T = (uint64_t)n_seq * S;
  if (int rc = make_tmap_bf16_2d(&m128, qkv, (uint64_t)3 * H * D, T, ld, 64, 128)) return rc;
  if (int rc = make_tmap_bf16_2d(&m64, qkv, (uint64_t)3 * H * D, T, ld, 64, 64)) return rc;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fwd_ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SMEM_BYTES);
    if (e != cudaSuccess) return set_cuda_error(e, "attn fwd_ts: cudaFuncSetAttribute");
    configured = true;
  }
  const int items = (S / BQ) * H * n_seq;
  const int slots = 2 * num_sms();
  const int grid = items < slots ? items : slots;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fwd_ts_kernel, m128, m64, (__nv_bfloat16*)out,
                                     (float*)lse, S, H, n_seq, scale);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn fwd_ts launch");
}
}  // namespace fa_ts

// ---------------------------------------------------------------- two query tiles per CTA
// One persistent CTA per SM processes PAIRS of query tiles (A = 2p, B = 2p+1) of one
// (head, sequence): the tensor core alternates between the tiles —
//   S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
// so while softmax warpgroup A works on S_A(j+1), the tensor core computes PV_B(j) and
// S_B(j+1), and vice versa.  P_X is written into the first columns of S_X (bf16
// pairs) and consumed from TMEM by the PV MMA; S_X(j+1) is issued after PV_X(j), and
// tcgen05 MMAs of one thread execute in order, so S_X(j+1) completing also means
// PV_X(j) consumed P_X(j) and O_X holds P_X(j) V_j (the rescale point).
// TMEM: S_A | S_B | O_A | O_B = 256 + 2D columns.  K/V blocks are shared by the two tiles.
namespace fa_pp {
constexpr int BQ = 128, BKV = 128;
// HV = softmax warps per TMEM lane quarter and tile (column halves of S / O)
template <int HV> constexpr int threads_for() { return 128 + 2 * 4 * HV * 32; }
constexpr float LOG2E = 1.4426950408889634f;
template <int D>
struct Smem {
  static constexpr int NST = (D == 64) ? 4 : 2;
  static constexpr int Q_BYTES = BQ * D * 2, KV_BYTES = BKV * D * 2;
  // Q tile pairs: double-buffered at D = 64, so the next item's Q is resident before
  // the current item's MMAs finish (D = 128: no room)
  static constexpr int QBUF = (D == 64) ? 2 : 1;
  __host__ __device__ static constexpr int off_q(int buf, int x) { return (buf * 2 + x) * Q_BYTES; }
  static constexpr int OFF_K = 2 * QBUF * Q_BYTES;
  static constexpr int OFF_V = OFF_K + NST * KV_BYTES;
  static constexpr int OFF_X = OFF_V + NST * KV_BYTES;  // [2 tiles][2 halves][128] exchange
  static constexpr int OFF_BAR = OFF_X + 2 * 2 * BQ * 4;
  static constexpr int TOTAL = OFF_BAR + 256 + 1024;
};

template <int D, int HV>
__global__ void __launch_bounds__(threads_for<HV>(), 1)
    fwd_pp_kernel(const __grid_constant__ CUtensorMap tm_rows128,
                  const __grid_constant__ CUtensorMap tm_rows64, __nv_bfloat16* __restrict__ out,
                  float* __restrict__ lse, int S, int H, int n_seq, float scale) {
  using L = Smem<D>;
  constexpr int NST = L::NST;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + L::OFF_BAR);
  constexpr int QBUF = L::QBUF;
  uint64_t* q_full = bar + 0;             // [QBUF]
  uint64_t* q_empty = bar + 2;            // [QBUF]
  uint64_t* kv_full = bar + 4;            // [NST]
  uint64_t* kv_empty = bar + 4 + NST;     // [NST]
  uint64_t* s_full = bar + 4 + 2 * NST;   // [2] per tile
  uint64_t* p_full = s_full + 2;          // [2] per tile (count 4)
  uint64_t* o_done = s_full + 4;          // [2] per tile: last PV of the item
  uint64_t* o_empty = s_full + 6;         // [2] per tile: epilogue read O (count 4)
  uint64_t* pv_done = s_full + 8;         // [2] per tile: each PV MMA complete (SEP)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 10);
  // SEP (D = 64): P is written to its own TMEM columns [384 + 64x, 448 + 64x) instead of
  // over S, so S_x(j+1) is issued as soon as the softmax of block j is done reading
  // S_x(j) — before PV_x(j) — and the next softmax waits one MMA less.  The softmax then
  // waits PV_x(j) (pv_done) before rescaling O or writing P(j+1).
  constexpr bool SEP = D == 64;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = S / (2 * BQ);
  const int HD = H * D;
  const int per_q = H * n_seq;
  const int items = npair * per_q;
  const int P = gridDim.x;
  auto item_of = [&](int k) { return k * P + ((k & 1) ? (P - 1 - (int)blockIdx.x) : (int)blockIdx.x); };
  auto decode = [&](int t, int& pr, int& h, int& b) {
    pr = npair - 1 - t / per_q;  // heavy pairs first
    const int rem = t % per_q;
    h = rem % H;
    b = rem / H;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_rows128);
    tma_prefetch_desc(&tm_rows64);
    for (int i = 0; i < QBUF; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < NST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 4 * HV);
      mbar_init(&o_done[x], 1);
      mbar_init(&o_empty[x], 4 * HV);
      mbar_init(&pv_done[x], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // PDL: prologue overlapped the previous kernel's tail
  griddep_launch();
  const uint32_t t_s[2] = {tmem, tmem + 128};
  const uint32_t t_o[2] = {tmem + 256, tmem + 256 + D};
  const uint32_t t_p[2] = {tmem + 384, tmem + 448};   // SEP only

  TR_DECL;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int g = 0, lt = 0;
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int pr, h, b;
        decode(t, pr, h, b);
        const int row0 = b * S, qa = 2 * pr, qb = qa + 1;
        TR_T0();
        const int qbuf = lt % QBUF;
        mbar_wait(&q_empty[qbuf], ((lt / QBUF) & 1) ^ 1);
        TR_ACC(0);
        mbar_arrive_expect_tx(&q_full[qbuf], 2 * L::Q_BYTES);
#pragma unroll
        for (int kc = 0; kc < D / 64; ++kc) {
          tma_load_2d(sm + L::off_q(qbuf, 0) + kc * BQ * 128, &tm_rows128, &q_full[qbuf],
                      h * D + kc * 64, row0 + qa * BQ);
          tma_load_2d(sm + L::off_q(qbuf, 1) + kc * BQ * 128, &tm_rows128, &q_full[qbuf],
                      h * D + kc * 64, row0 + qb * BQ);
        }
        for (int j = 0; j <= qb; ++j, ++g) {
          const int st = g % NST;
          TR_T0();
          mbar_wait(&kv_empty[st], ((g / NST) & 1) ^ 1);
          TR_ACC(1);
          mbar_arrive_expect_tx(&kv_full[st], 2 * L::KV_BYTES);
          uint8_t* kd = sm + L::OFF_K + st * L::KV_BYTES;
          uint8_t* vd = sm + L::OFF_V + st * L::KV_BYTES;
          const int kr = row0 + j * BKV;
#pragma unroll
          for (int kc = 0; kc < D / 64; ++kc)
            tma_load_2d(kd + kc * BKV * 128, &tm_rows128, &kv_full[st], HD + h * D + kc * 64, kr);
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
#pragma unroll
            for (int dc = 0; dc < D / 64; ++dc)
              tma_load_2d(vd + (kb * (D / 64) + dc) * 8192, &tm_rows64, &kv_full[st],
                          2 * HD + h * D + dc * 64, kr + kb * 64);
        }
      }
      TR_PRINT("tma", 0);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(BQ, BKV, 0, 0);
      constexpr uint32_t idesc_o = umma_idesc_bf16(BQ, D, 0, 1);
      const uint32_t ts0 = tmem, ts1 = tmem + 128, to0 = tmem + 256, to1 = tmem + 256 + D;
      const uint32_t tp0 = tmem + 384, tp1 = tmem + 448;
      int g = 0, lt = 0;
      int ns0 = 0, ns1 = 0;  // S blocks issued per tile (parity of p_full waits)
      bool s0_next = false;  // the next item's S_0(0) was issued early (SEP)
      // (tile index x is a compile-time constant in every call below: no
      // dynamically indexed local arrays on the issue path)
      for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
        int pr, h, b;
        decode(t, pr, h, b);
        const int qa = 2 * pr, qb = qa + 1;
        const int qbuf = lt % QBUF;
        mbar_wait(&q_full[qbuf], (lt / QBUF) & 1);
        // S_x(j) = Q_x K_j^T for the item whose Q sits in buffer qbf and whose K/V blocks
        // start at ring position gb
        auto issue_s_at = [&](auto xc, int j, int qbf, int gb) {
          constexpr int x = decltype(xc)::value;
          const int st = (gb + j) % NST;
          TR_T0();
          mbar_wait(&kv_full[st], ((gb + j) / NST) & 1);
          TR_ACC(0);
          tc_fence_after();
          const uint32_t k_base = smem_u32(sm + L::OFF_K + st * L::KV_BYTES);
          const uint32_t qb_ = smem_u32(sm + L::off_q(qbf, x));
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            mma_bf16_ss(x ? ts1 : ts0, desc_kmajor(qb_, kk, BQ), desc_kmajor(k_base, kk, BKV),
                        idesc_s, kk > 0 ? 1u : 0u);
          mma_commit(&s_full[x]);
        };
        auto issue_s = [&](auto xc, int j) { issue_s_at(xc, j, qbuf, g); };
        auto issue_pv = [&](auto xc, int j) {  // O_x += P_x(j) V_j, P_x from TMEM
          constexpr int x = decltype(xc)::value;
          const int st = (g + j) % NST;
          int& ns = x ? ns1 : ns0;
          mbar_wait(&p_full[x], ns & 1);
          ++ns;
          TR_T0();
          if (j == 0) mbar_wait(&o_empty[x], (lt & 1) ^ 1);
          TR_ACC(2);
          tc_fence_after();
          const uint32_t v_base = smem_u32(sm + L::OFF_V + st * L::KV_BYTES);
          const uint32_t tsx = x ? ts1 : ts0, tox = x ? to1 : to0;
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t bdesc = umma_desc_sw128(
                v_base + (kk >> 2) * (D / 64) * 8192 + (kk & 3) * 2048, 8192, 1024);
            // P keys [64h, 64h+64) sit in the S columns of half h (see the softmax), or
            // contiguously in the tile's own P columns (SEP)
            const uint32_t a_tm = SEP ? (x ? tp1 : tp0) + kk * 8
                                      : (HV == 2 ? tsx + (kk >> 2) * 64 + (kk & 3) * 8 : tsx + kk * 8);
            mma_bf16_ts(tox, a_tm, bdesc, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (SEP) mma_commit(&pv_done[x]);
          if (j == (x ? qb : qa)) mma_commit(&o_done[x]);
        };
        using X0 = std::integral_constant<int, 0>;
        using X1 = std::integral_constant<int, 1>;
        if (!s0_next) issue_s(X0{}, 0);
        s0_next = false;
        issue_s(X1{}, 0);
        for (int j = 0; j <= qb; ++j) {
          if constexpr (SEP) {
            // S_x(j+1) right after the softmax released S_x(j) (p_full), then PV_x(j)
            if (j <= qa) {
              TR_T0();
              mbar_wait(&p_full[0], ns0 & 1);
              TR_ACC(1);
              if (j + 1 <= qa) issue_s(X0{}, j + 1);
              issue_pv(X0{}, j);
            }
            if (j == qb && QBUF == 2 && item_of(k + 1) < items) {
              // tile 0 is done with this item: start the next item's S_0(0) now, while
              // tile 1 finishes its last (diagonal) block
              const int nbuf = (lt + 1) % QBUF;
              mbar_wait(&q_full[nbuf], ((lt + 1) / QBUF) & 1);
              issue_s_at(X0{}, 0, nbuf, g + qb + 1);
              s0_next = true;
            }
            TR_T0();
            mbar_wait(&p_full[1], ns1 & 1);
            TR_ACC(1);
            if (j + 1 <= qb) issue_s(X1{}, j + 1);
            issue_pv(X1{}, j);
            mma_commit(&kv_empty[(g + j) % NST]);  // K_j, V_j no longer read
          } else {
            if (j <= qa) {
              issue_pv(X0{}, j);
              if (j + 1 <= qa) issue_s(X0{}, j + 1);
            }
            issue_pv(X1{}, j);
            mma_commit(&kv_empty[(g + j) % NST]);  // K_j, V_j no longer read
            if (j + 1 <= qb) issue_s(X1{}, j + 1);
          }
        }
        mma_commit(&q_empty[qbuf]);
        g += qb + 1;
      }
      TR_PRINT("mma", 0);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax: per tile, 4*HV warps
    // (warp -> TMEM lane quarter wq and column half hf; with HV == 2 the halves
    // exchange row maxima / sums through smem with a 64-thread named barrier and each
    // half writes its P columns into its own S columns: keys [64h, 64h+64) -> S
    // columns [64h, 64h+32))
    const int idx = warp - 4;
    const int x = idx / (4 * HV);
    const int sub = idx % (4 * HV);
    const int wq = sub & 3, hf = HV == 2 ? (sub >> 2) : 0;
    const int r = wq * 32 + lane;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const float sl2 = scale * LOG2E;
    constexpr float RESCALE_T = 8.f;
    constexpr int NCH = (BKV / 32) / HV;  // 32-column S chunks per warp
    const uint32_t ts = x ? t_s[1] : t_s[0], to = x ? t_o[1] : t_o[0];
    const uint32_t tp = x ? t_p[1] : t_p[0];
    int npv = 0;  // PV MMAs of this tile issued before the current block (SEP)
    float* xch = reinterpret_cast<float*>(sm + L::OFF_X) + x * 2 * BQ;
    auto pair_sync = [&]() {
      if constexpr (HV == 2) asm volatile("bar.sync %0, 64;" ::"r"(1 + x * 4 + wq) : "memory");
    };
    // ALT: the exponential passes of tile 0 and tile 1 take turns (named barriers E0 / E1,
    // both tiles' softmax warps), so one tile's S wait / row max / rescale overlap the
    // other tile's MUFU-bound pass instead of both tiles contending for the MUFU at once.
    // Per item tile 0 runs qa+1 passes and tile 1 qa+2: order T0(0) T1(0) ... T0(qa)
    // T1(qa) T1(qb); T1(qb) hands over to the next item's T0(0).
    constexpr int kAltE0 = 9, kAltE1 = 10, kAltN = 2 * 4 * HV * 32;
    auto alt_sync = [&](int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kAltN) : "memory"); };
    auto alt_arrive = [&](int id) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(kAltN) : "memory"); };
    int nb = 0, lt = 0;  // S blocks consumed by this tile (s_full parity)
    for (int k = 0, t = item_of(0); t < items; t = item_of(++k), ++lt) {
      int pr, h, b;
      decode(t, pr, h, b);
      const int qx = 2 * pr + x;             // this warpgroup's query tile
      const bool last_item = item_of(k + 1) >= items;
      const int row0 = b * S;
      const int q = qx * BQ + r;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j <= qx; ++j) {
        const bool diag = j == qx;
        TR_T0();
        mbar_wait(&s_full[x], nb & 1);
        ++nb;
        tc_fence_after();
        TR_ACC(0);
        // The warp's S columns are read as 16-column sub-chunks, software-pipelined: the
        // load of sub-chunk sc+1 is in flight while sub-chunk sc is processed (one
        // tcgen05.wait::ld per sub-chunk covers it).
        constexpr int NS16 = 2 * NCH;
        const uint32_t s_cols = ts + lane_off + hf * NCH * 32;
        const int col0 = hf * NCH * 32;
        auto s_pass = [&](auto&& proc) {
          uint32_t va[16], vb[16];
          tmem_ld_32x32b_x16(s_cols, va);
          tmem_ld_wait_regs16(va);
#pragma unroll
          for (int sc = 0; sc < NS16; sc += 2) {
            tmem_ld_32x32b_x16(s_cols + (sc + 1) * 16, vb);
            proc(va, sc);
            tmem_ld_wait_regs16(vb);
            if (sc + 2 < NS16) tmem_ld_32x32b_x16(s_cols + (sc + 2) * 16, va);
            proc(vb, sc + 1);
            if (sc + 2 < NS16) tmem_ld_wait_regs16(va);
          }
        };
        auto row_max = [&](auto diag_c) {
          constexpr bool DG = decltype(diag_c)::value;
          float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
          s_pass([&](const uint32_t (&v)[16], int sc) {
            float xs[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              xs[i] = __uint_as_float(v[i]);
              if (DG && col0 + sc * 16 + i > r) xs[i] = -INFINITY;
            }
#pragma unroll
            for (int i = 0; i < 16; i += 8) {
              mx4[0] = fmax3(mx4[0], xs[i], xs[i + 1]);
              mx4[1] = fmax3(mx4[1], xs[i + 2], xs[i + 3]);
              mx4[2] = fmax3(mx4[2], xs[i + 4], xs[i + 5]);
              mx4[3] = fmax3(mx4[3], xs[i + 6], xs[i + 7]);
            }
          });
          return fmaxf(fmax3(mx4[0], mx4[1], mx4[2]), mx4[3]);
        };
        // exponentials with the running max m; P lands in the tile's P columns (SEP) or
        // inside this warp's own (already read) S columns
        auto exp_pack = [&](auto diag_c) {
          constexpr bool DG = decltype(diag_c)::value;
          float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-m, -m);
          s_pass([&](const uint32_t (&v)[16], int sc) {
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float2 e = ffma2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])),
                                     sl2x2, nm2);
              float p0 = exp2_fast(e.x);
              float p1 = exp2_fast(e.y);
              if (DG && col0 + sc * 16 + i > r) p0 = 0.f;
              if (DG && col0 + sc * 16 + i + 1 > r) p1 = 0.f;
              rs2[(i >> 1) & 1] = fadd2(rs2[(i >> 1) & 1], make_float2(p0, p1));
              pk[i >> 1] = pack_bf16(p0, p1);
            }
            if constexpr (SEP)
              tmem_st_32x32b_x8(tp + lane_off + hf * 32 + sc * 8, pk);
            else
              tmem_st_32x32b_x8(ts + lane_off + hf * 64 + sc * 8, pk);
          });
          return (rs2[0].x + rs2[1].x) + (rs2[0].y + rs2[1].y);
        };
        auto exchange_max = [&](float mh) {
          if constexpr (HV == 2) {
            xch[hf * BQ + r] = mh;
            pair_sync();
            mh = fmaxf(mh, xch[(hf ^ 1) * BQ + r]);
            pair_sync();
          }
          return mh;
        };
        auto rescale_o = [&](float corr) {  // O holds P(j-1) V_{j-1} (see above)
#pragma unroll
          for (int c = hf * (D / 32 / HV); c < (hf + 1) * (D / 32 / HV); ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(to + lane_off + c * 32, v);
            tmem_ld_wait_regs(v);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(to + lane_off + c * 32, v);
          }
        };
        // exponential passes of the two tiles alternate (see ALT above)
        auto alt_enter = [&]() {
          if constexpr (!SEP) return;
          if (x == 0 && !(k == 0 && j == 0)) alt_sync(kAltE0);
          if (x == 1 && j < qx) alt_sync(kAltE1);
        };
        auto alt_leave = [&]() {
          if constexpr (!SEP) return;
          if (x == 0) alt_arrive(kAltE1);
          if (x == 1 && (j < qx - 1 || (j == qx && !last_item))) alt_arrive(kAltE0);
        };
        float mh = diag ? row_max(std::true_type{}) : row_max(std::false_type{});
        TR_ACC(1);
        mh = exchange_max(mh);
        TR_ACC(2);
        if constexpr (SEP) {  // PV(previous block) complete: O may be rescaled, P rewritten
          if (npv > 0) mbar_wait(&pv_done[x], (npv - 1) & 1);
          ++npv;
          tc_fence_after();
        }
        TR_ACC(3);
        const float mx = mh * sl2;
        const bool move = mx > m + RESCALE_T;
        const float m_new = move ? mx : m;
        const float corr = move ? exp2_fast(m - m_new) : 1.f;
        m = m_new;
        if (j > 0 && __any_sync(0xffffffffu, move)) rescale_o(corr);
        TR_ACC(4);
        alt_enter();
        TR_ACC(6);
        const float rs = diag ? exp_pack(std::true_type{}) : exp_pack(std::false_type{});
        alt_leave();
        l = l * corr + rs;
        TR_ACC(5);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
        TR_ACC(7);
        TR_N();
      }
      // epilogue
      TR_T0();
      float lt_sum = l;
      if constexpr (HV == 2) {
        xch[hf * BQ + r] = l;
        pair_sync();
        lt_sum = l + xch[(hf ^ 1) * BQ + r];
        pair_sync();
      }
      TR_ACC(8);
      mbar_wait(&o_done[x], lt & 1);
      tc_fence_after();
      TR_ACC(9);
      const float inv = 1.f / lt_sum;
      __nv_bfloat16* orow = out + ((size_t)row0 + q) * HD + h * D;
      const bool st256 = ((reinterpret_cast<uintptr_t>(out) | (HD * 2)) & 31) == 0;
#pragma unroll
      for (int c = hf * (D / 32 / HV); c < (hf + 1) * (D / 32 / HV); ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(to + lane_off + c * 32, v);
        tmem_ld_wait_regs(v);
        TR_ACC(11);
#pragma unroll
        for (int i = 0; i < 32; i += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            pk[e] = pack_bf16(__uint_as_float(v[i + 2 * e]) * inv, __uint_as_float(v[i + 2 * e + 1]) * inv);
          if (st256) {
            st_global_256(orow + c * 32 + i, pk);
          } else {
            *reinterpret_cast<uint4*>(orow + c * 32 + i) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            *reinterpret_cast<uint4*>(orow + c * 32 + i + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
      }
      TR_ACC(12);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[x]);
      if (hf == 0) lse[((size_t)b * H + h) * S + q] = (m + __log2f(lt_sum)) * (1.f / LOG2E);
      TR_ACC(10);
    }
    if (r == 0 && hf == 0) TR_PRINT("softmax", x);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

template <int D, int HV>
static int run(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int ld, float scale,
               cudaStream_t s) {
  CUtensorMap m128, m64;
  const uint64_t T = (uint64_t)n_seq * S;
  if (int rc = make_tmap_bf16_2d(&m128, qkv, (uint64_t)3 * H * D, T, ld, 64, 128)) return rc;
  if (int rc = make_tmap_bf16_2d(&m64, qkv, (uint64_t)3 * H * D, T, ld, 64, 64)) return rc;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fwd_pp_kernel<D, HV>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<D>::TOTAL);
    if (e != cudaSuccess) return set_cuda_error(e, "attn fwd_pp: cudaFuncSetAttribute");
    configured = true;
  }
  const int items = (S / (2 * BQ)) * H * n_seq;
  const int grid = items < num_sms() ? items : num_sms();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads_for<HV>());
  cfg.dynamicSmemBytes = Smem<D>::TOTAL;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fwd_pp_kernel<D, HV>, m128, m64, (__nv_bfloat16*)out,
                                     (float*)lse, S, H, n_seq, scale);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn fwd_pp launch");
}
}  // namespace fa_pp

template <int D>
static int run_fwd(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int ld,
                   float scale, cudaStream_t s) {
  CUtensorMap m128, m64;
  const uint64_t T = (uint64_t)n_seq * S;
  if (int rc = make_tmap_bf16_2d(&m128, qkv, (uint64_t)3 * H * D, T, ld, 64, 128)) return rc;
  if (int rc = make_tmap_bf16_2d(&m64, qkv, (uint64_t)3 * H * D, T, ld, 64, 64)) return rc;
  const int smem = FwdSmem<D>::TOTAL;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "attn_sm100: cudaFuncSetAttribute");
    configured = true;
  }
  const int items = (S / BQ) * H * n_seq;
  const int grid = items < num_sms() ? items : num_sms();
  fwd_kernel<D><<<grid, kThreads, smem, s>>>(m128, m64, (__nv_bfloat16*)out, (float*)lse, S, H,
                                             n_seq, scale);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : set_cuda_error(e, "attn_sm100 fwd launch");
}

}  // namespace fa
}  // namespace zb

using namespace zb;

extern "C" int zb_attn_fwd(const void* qkv, void* out, void* lse, int n_seq, int S, int H,
                           int D, int ld, float scale, cudaStream_t s) {
  if (S % 128) return set_error(ZB_ERR_INVALID, "attn_fwd: seq_len must be a multiple of 128");
  if (ld % 8 || ((uintptr_t)qkv & 15)) return set_error(ZB_ERR_INVALID, "attn_fwd: bad ld/alignment");
  if (n_seq <= 0) return 0;
  // Pairs of query tiles per CTA when S % 256 == 0; else the two-CTA-per-SM kernel
  // (D = 64) / the single-tile kernel (D = 128).
  if (S % 256 == 0 && D == 64) return fa::fa_pp::run<64, 2>(qkv, out, lse, n_seq, S, H, ld, scale, s);
  if (S % 256 == 0 && D == 128) return fa::fa_pp::run<128, 1>(qkv, out, lse, n_seq, S, H, ld, scale, s);
  if (D == 64) return fa::fa_ts::run(qkv, out, lse, n_seq, S, H, ld, scale, s);
  if (D == 128) return fa::run_fwd<128>(qkv, out, lse, n_seq, S, H, ld, scale, s);
  return set_error(ZB_ERR_UNSUPPORTED, "attn_fwd: head_dim %d unsupported (64, 128)", D);
}
