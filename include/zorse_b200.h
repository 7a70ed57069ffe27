/*
 * zorse_b200.h — C ABI of libzorse_b200.so, the B200 (sm_100a) executor of the
 * Zorse training-step hot path.
 *
 * The reference (hetplan, arXiv 2507.10392) has no runtime: every hot-path
 * operation is a MODELLED task in its discrete-event simulator.  Each entry
 * point below is the real operation behind one of those tasks; the comment on
 * each names the reference task / formula it replaces (paths relative to
 * /root/reference/pkg/src/hetplan/).
 *
 * Conventions
 *   - Every function returns 0 on success, a nonzero code otherwise
 *     (1001 invalid argument, 1002 CUDA error, 1003 NCCL error, 1004
 *     unsupported shape); zb_last_error() gives a thread-local message.
 *   - The caller owns all device memory; the library allocates nothing on the
 *     hot path.  Pointers are device pointers unless stated otherwise.
 *   - Every kernel is enqueued on the given stream; no call synchronises.
 *   - bf16 = IEEE bfloat16, fp32 accumulators; matrices are row-major with the
 *     given leading dimension (elements).
 *   - There is no CPU fallback: without a B200 these calls fail.
 */
#ifndef ZORSE_B200_H
#define ZORSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* zb_stream_t; /* == cudaStream_t */

/* ---------------------------------------------------------------- status */
const char* zb_last_error(void);
int zb_version(void);
int zb_device_sync(void);

/* ---------------------------------------------------------------- GEMM
 * C[M,N] = A[M,K] * B[N,K]^T on tcgen05 tensor cores (TMA-fed, TMEM accumulators).
 * a_mn_major: A stored [K][lda] (M contiguous) instead of [M][lda].
 * b_mn_major: B stored [K][ldb] (N contiguous) instead of [N][ldb].
 * epilogue: 0 C=acc | 1 C=acc+bias | 2 aux=acc+bias, C=gelu(aux) | 3 C=acc+bias+R
 *           4 C=acc*gelu'(aux) | 5 C(fp32)=beta*C+acc | 6 C=acc+R | 7 C=gelu(acc+bias) (no aux)
 * Replaces the modelled per-layer compute of Fwd / Recompute / Bwd tasks
 * (simulate.py:330-367, 469-505; compute_time simulate.py:177-195). */
int zb_gemm_bf16(const void* A, const void* B, void* C, const void* bias, const void* R,
                 void* aux, int M, int N, int K, int lda, int ldb, int ldc, int ldr, int ldaux,
                 int a_mn_major, int b_mn_major, int epilogue, float beta, zb_stream_t stream);
/* The tile zb_gemm_bf16 picks: the committed B200 tile table (gemm_tune_cache.txt
 * beside the library, read once, never written by the library), else the wave-
 * quantisation cost model.  pair: 0 1-CTA 128xBN, 1 CTA pair 256xBN, 2 two pairs
 * multicasting A; bn 128/192/256; splits = K splits (fp32 beta=1 accumulation only). */
int zb_gemm_choice(int M, int N, int K, int a_mn_major, int b_mn_major, int epilogue,
                   float beta, int ldc, int* pair, int* bn, int* splits, int* from_table);
/* zb_gemm_bf16 with an explicit tile (tests, benchmarks, tuning); a negative pair /
 * raster or a zero bn / splits keeps the default for that field.  raster: 0 M-fastest,
 * 1 N-fastest tile order.  tma_epi = 0 forces the direct-store epilogue. */
int zb_gemm_bf16_tile(const void* A, const void* B, void* C, const void* bias, const void* R,
                      void* aux, int M, int N, int K, int lda, int ldb, int ldc, int ldr,
                      int ldaux, int a_mn_major, int b_mn_major, int epilogue, float beta,
                      int pair, int bn, int splits, int raster, int tma_epi, zb_stream_t stream);
/* Times the cost model's tile and its neighbours on scratch outputs (inputs only read)
 * and returns the fastest.  Synchronises `stream`; rejected during graph capture.
 * Offline tuning only (scripts/tune_gemm.py writes the tile table). */
int zb_gemm_tune(const void* A, const void* B, const void* bias, const void* R, void* aux,
                 int M, int N, int K, int lda, int ldb, int ldc, int ldr, int ldaux,
                 int a_mn_major, int b_mn_major, int epilogue, float beta, int* pair, int* bn,
                 int* splits, zb_stream_t stream);

/* ---------------------------------------------------------------- attention
 * Causal attention over the fused QKV rows ([q|k|v] per token, pitch ld),
 * n_seq sequences of S tokens (S % 128 == 0), H heads of dim D (64 or 128), on
 * 5th-gen tensor cores: S and O accumulate in TMEM, Q/K/V tiles streamed by TMA.
 * out [n_seq*S, H*D] bf16; lse [n_seq, H, S] fp32.  Same tasks as above. */
int zb_attn_fwd(const void* qkv, void* out, void* lse, int n_seq, int S, int H, int D, int ld,
                float scale, zb_stream_t stream);
/* Writes dQ, dK, dV into the matching columns of dqkv (pitch ld); dout pitch H*D,
 * 16-byte aligned.  delta: fp32 scratch [n_seq, H, S].  With dq_accum (fp32
 * [n_seq*S][H*D] workspace) and D == 64: one fused pass (dQ partials reduce-added into
 * dq_accum, then scaled into dqkv); otherwise two passes (dK/dV, then dQ) without
 * atomics. */
int zb_attn_bwd(const void* qkv, const void* out, const void* dout, const void* lse, void* dqkv,
                void* dq_accum, void* delta, int n_seq, int S, int H, int D, int ld, float scale,
                zb_stream_t stream);

/* ---------------------------------------------------------------- elementwise
 * LayerNorm over rows of length d (d % 8 == 0).  mean/rstd: fp32 [rows]. */
int zb_layernorm_fwd(const void* x, const void* w, const void* b, void* y, void* mean, void* rstd,
                     void* reserved, int rows, int d, float eps, zb_stream_t stream);
/* dx = dres + LN'(dy) (dres may be NULL; dx may alias dres but not dy or x); dw, db (fp32) += grads.
 * Two launches: dx per row, then the dw / db column reduction. */
int zb_layernorm_bwd(const void* dy, const void* x, const void* w, const void* mean,
                     const void* rstd, void* dx, void* dw, void* db, const void* dres, int rows,
                     int d, zb_stream_t stream);
/* Same, and (db_res, db_out non-NULL, dres required) the column sums of dres and of the
 * dx output accumulated into db_res / db_out: the bias gradients of the linear layers
 * whose output gradients they are (GPT block: fc2 and the attention projection),
 * folded into the dw / db column pass instead of two zb_bias_grad launches. */
int zb_layernorm_bwd_ex(const void* dy, const void* x, const void* w, const void* mean,
                        const void* rstd, void* dx, void* dw, void* db, const void* dres,
                        void* db_res, void* db_out, int rows, int d, zb_stream_t stream);
/* zb_layernorm_bwd_ex split in its two launches: phase 1 = dx only, phase 2 = the dw / db
 * (and db_res / db_out) column pass only, which reads dx — the caller orders phase 2 after
 * phase 1 (e.g. on a second stream behind an event); phase 0 = both. */
int zb_layernorm_bwd_phase(const void* dy, const void* x, const void* w, const void* mean,
                           const void* rstd, void* dx, void* dw, void* db, const void* dres,
                           void* db_res, void* db_out, int rows, int d, int phase,
                           zb_stream_t stream);
/* out[t] = wte[tok[t]] + wpe[t % seq]  (tok: int32; wpe may be NULL). */
int zb_embedding_fwd(const void* tok, const void* wte, const void* wpe, void* out, int rows, int d,
                     int seq, zb_stream_t stream);
/* dwte[tok[t]] += dout[t]; dwpe[t % seq] += dout[t]  (fp32 accumulators). */
int zb_embedding_bwd(const void* tok, const void* dout, void* dwte, void* dwpe, int rows, int d,
                     int seq, zb_stream_t stream);
/* Fused softmax cross-entropy: *loss_sum += sum_rows (lse - logit[label]);
 * dlogits = (softmax - onehot) * scale (may alias logits); label < 0 ignores a row. */
int zb_xent_fwd_bwd(const void* logits, const void* labels, void* loss_sum, void* dlogits,
                    int rows, int V, int ld, float scale, zb_stream_t stream);
/* db[n] (fp32) += sum_rows dy[row, n]. */
int zb_bias_grad(const void* dy, void* db, int rows, int n, int ld, zb_stream_t stream);
/* Llama family: RMSNorm (rstd fp32 [rows]); dw (fp32) += grad; dres may be NULL. */
int zb_rmsnorm_fwd(const void* x, const void* w, void* y, void* rstd, int rows, int d, float eps,
                   zb_stream_t stream);
int zb_rmsnorm_bwd(const void* dy, const void* x, const void* w, const void* rstd, void* dx,
                   void* dw, const void* dres, int rows, int d, zb_stream_t stream);
/* Rotary embedding in place on the q and k parts of fused QKV rows (pitch ld,
 * rotate-half pairs (i, i+D/2), angle pos*theta^(-2i/D), pos = row % S);
 * inverse=1 applies the transpose rotation (gradient). */
int zb_rope(void* qkv, int rows, int S, int H, int D, int ld, float theta, int inverse,
            zb_stream_t stream);
/* gu rows = [gate(f) | up(f)]: out = silu(gate)*up; backward writes [dgate | dup] (may alias gu). */
int zb_swiglu_fwd(const void* gu, void* out, int rows, int f, zb_stream_t stream);
int zb_swiglu_bwd(const void* gu, const void* dout, void* dgu, int rows, int f, zb_stream_t stream);
int zb_cast_f32_bf16(const void* src, void* dst, int64_t n, zb_stream_t stream);
int zb_fill_f32(void* p, float value, int64_t n, zb_stream_t stream);
int zb_add_bf16(const void* a, const void* b, void* out, int64_t n, zb_stream_t stream);

/* ---------------------------------------------------------------- optimizer
 * Fused AdamW on one rank's uneven fp32 shard; writes the bf16 parameter shard.
 * sumsq (fp32 scalar, may be NULL) += sum (grad*grad_scale)^2.
 * Replaces the OptimStep task (simulate.py:536-550; optim_update_per_param costs.py:81). */
int zb_adamw_shard(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                   void* param_bf16, void* sumsq, int64_t n, float lr, float beta1, float beta2,
                   float eps, float weight_decay, float grad_scale, int step, zb_stream_t stream);

/* Same, with the step number t read from device memory (*step_dev, int32) so a
 * captured CUDA graph replays correct bias corrections; zb_step_increment adds 1. */
int zb_adamw_shard_dstep(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                         void* param_bf16, void* sumsq, int64_t n, float lr, float beta1,
                         float beta2, float eps, float weight_decay, float grad_scale,
                         const void* step_dev, zb_stream_t stream);
/* Row-split update of a [rows, d] embedding table whose gradient is nonzero only in the
 * rows of this step's tokens.  zb_embed_mark: mark[tok] = *stamp_dev (the device step
 * counter) for every token.  zb_embed_zero_rows: grad rows of the tokens <- 0.
 * zb_adamw_rows_dstep: AdamW over the rows with (mark[r] == *step_dev) == marked; marked = 0
 * updates with g = 0 and reads no gradient (grad may be NULL).  Per element identical to
 * zb_adamw_shard_dstep with a zero gradient in the unmarked rows. */
int zb_embed_mark(const void* tokens, int64_t n, int rows, void* mark, const void* stamp_dev,
                  zb_stream_t stream);
int zb_embed_zero_rows(const void* tokens, int64_t n, int rows, void* grad, int d,
                       zb_stream_t stream);
int zb_adamw_rows_dstep(void* master, void* exp_avg, void* exp_avg_sq, const void* grad,
                        void* param_bf16, void* sumsq, int rows, int d, const void* mark,
                        int marked, float lr, float beta1, float beta2, float eps,
                        float weight_decay, float grad_scale, const void* step_dev,
                        zb_stream_t stream);
int zb_step_increment(void* step_dev, zb_stream_t stream);

/* ---------------------------------------------------------------- collectives
 * Communicators are opaque NCCL handles owned by the executor. dtype: 0 bf16, 1 fp32. */
int zb_nccl_unique_id_size(void);
int zb_nccl_get_unique_id(void* out /* host, zb_nccl_unique_id_size() bytes */);
int zb_comm_init(void** comm_out, const void* unique_id /* host */, int nranks, int rank);
int zb_comm_destroy(void* comm);
/* Uneven in-place AllGather of a flat buffer: rank r's shard is
 * buf[displs[r] : displs[r]+counts[r]] (counts/displs: host int64 arrays).
 * Replaces the AllGather task (simulate.py:292-328, 408-446; costs.py:138-149). */
int zb_allgather_v(void* comm, void* buf, const int64_t* counts, const int64_t* displs,
                   int nranks, int dtype, zb_stream_t stream);
/* Uneven in-place ReduceScatter (sum): afterwards rank r's slice holds the group sum.
 * Replaces the ReduceScatter task (simulate.py:523-534; costs.py:152-158). */
int zb_reduce_scatter_v(void* comm, void* buf, const int64_t* counts, const int64_t* displs,
                        int nranks, int dtype, zb_stream_t stream);
/* Grouped point-to-point transfers (world ranks); stage-boundary activations and
 * gradients.  Replaces P2PSend / P2PRecv (simulate.py:378-385, 507-514; costs.py:161-186). */
int zb_p2p_group(void* comm, int n, const int* peers, void* const* bufs, const int64_t* counts,
                 const int* is_send, int dtype, zb_stream_t stream);
int zb_allreduce_sum(void* comm, void* buf, int64_t count, int dtype, zb_stream_t stream);

/* ---- NVLink peer-memory collectives of one DP group (csrc/peer.cu) ------------------
 * Each rank exports one arena with a CUDA IPC handle: per parameter unit a 16-byte
 * flag record {param_ready, grad_ready, done, pad} (same offset on every rank), the
 * fp32 gradient window slots (same offsets on every rank) and the rank's persistent
 * bf16 parameter shard (rank-specific offset).  `bases[p]` is rank p's arena base
 * as mapped in this process (bases[me] local).  Offsets are byte offsets. */
int zb_ipc_handle_size(void);
int zb_ipc_get_handle(const void* ptr, void* handle_out, uint64_t* offset_out);
int zb_ipc_open(const void* handle, void** base_out);
int zb_ipc_close(void* base);
/* *flag = *epoch_dev + delta with system-scope release (after a system fence). */
int zb_peer_signal(void* flag, const void* epoch_dev, int delta, zb_stream_t stream);
/* Single-process multi-GPU (tests, NVLink probes): enable the current device's
 * access to peer_device's memory (cudaDeviceEnablePeerAccess; idempotent). */
int zb_peer_enable(int peer_device);
/* Bound of every flag spin (seconds; 0 = unbounded; default 120).  A spin that
 * exceeds it prints the flag it waited for and traps. */
int zb_peer_set_timeout(double seconds);
/* One-CTA kernel: wait until every peer's flag at flag_off >= *epoch_dev + delta
 * (e.g. param_ready of a unit: the peers finished reading its gradient slot). */
int zb_peer_wait(void* const* bases, int nranks, int me, uint64_t flag_off,
                 const void* epoch_dev, int epoch_delta, zb_stream_t stream);
/* AllGather-v before a layer (replaces the AllGather task, simulate.py:292-328 and
 * :408-446; costs.py:138-149): wait for every peer's param_ready >= *epoch_dev +
 * epoch_delta, then copy rank p's shard (counts[p] elements at bases[p] +
 * shard_offs[p]) to dst + displs[p] (local full buffer) for every p.  mode 0: copy
 * engines; mode 1: SM pull kernel. */
int zb_peer_allgather_v(void* const* bases, int nranks, int me, const uint64_t* shard_offs,
                        void* dst, int elem_bytes, const int64_t* counts, const int64_t* displs,
                        uint64_t flag_off, const void* epoch_dev, int epoch_delta, int mode,
                        zb_stream_t stream);
/* ReduceScatter-v + grad scale + AdamW + bf16 cast in one kernel (replaces the
 * ReduceScatter task simulate.py:523-534 followed by OptimStep :536-550): publish
 * grad_ready = *epoch_dev, wait for all peers', sum the fp32 gradient slices
 * [lo, lo+n) of every peer's grad buffer (grad_off), update master / exp_avg /
 * exp_avg_sq (torch AdamW), write the bf16 shard to param_bf16 and (if non-NULL) the
 * reduced gradient to grad_out, accumulate sum(g^2) into sumsq (if non-NULL); the
 * last CTA publishes param_ready = *epoch_dev. */
int zb_peer_rs_adamw(void* const* bases, int nranks, int me, uint64_t grad_off, int64_t lo,
                     int64_t n, uint64_t flag_off, const void* epoch_dev, void* master,
                     void* exp_avg, void* exp_avg_sq, void* param_bf16, void* grad_out,
                     void* sumsq, float lr, float beta1, float beta2, float eps,
                     float weight_decay, float grad_scale, const void* step_dev,
                     zb_stream_t stream);

/* ---- host: planner min-cut kernel (csrc/mincut.cpp) ---------------------------------
 * Global minimum 2-cut of a dense symmetric float64 [n][n] graph (Stoer-Wagner),
 * ties toward the smallest lexrank; bit-identical to the reference's only FFI,
 * hetplan `min_cut_kernel(weights, lexrank) -> (float, sorted list[int])`
 * (_mincut_c.pyx:16-82, bound at partition.py:26-38).  side_out must hold n entries;
 * *side_len receives the size of the returned (sorted) shore. */
int zb_min_cut(const double* weights, int64_t n, const int64_t* lexrank, double* cut_out,
               int64_t* side_out, int64_t* side_len);

/* ---- host: planner Eq.1 latency (csrc/eq1.cpp) ---------------------------------------
 * Iteration latency of one candidate plan — the planner's hot loop (costs.py:204-535:
 * _compute_per_microbatch :220-249, phase recurrence :323-360, total_iteration_latency
 * :384-535), bit-identical to the Python restatement.  n ministages in global order:
 * grp[s], q[s] (group, round); layer classes of stage s = lay_cls[lay_off[s] ..
 * lay_off[s+1]); distinct (kind, share > 0) members of its group = mem_kind / mem_share
 * [mem_off[s] .. mem_off[s+1]); fits[(kind * n_cls + cls) * 4 + {fwd_alpha, fwd_beta,
 * bwd_alpha, bwd_beta}]; ag / rs / p2p / stage_params per stage (summed AllGather,
 * ReduceScatter, incoming boundary transfer time, parameter count); group_size per
 * group.  out = {l_forwards, l_backwards, l_startup}. */
int zb_eq1_latency(int n, int m, int z3, int offloads, int rounds, const int* grp, const int* q,
                   const int* lay_off, const int* lay_cls, const int* mem_off,
                   const int* mem_kind, const int* mem_share, int n_cls, const double* fits,
                   const double* ag, const double* rs, const double* p2p,
                   const double* stage_params, int n_groups, const int* group_size,
                   double optim_per_param, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ZORSE_B200_H */
