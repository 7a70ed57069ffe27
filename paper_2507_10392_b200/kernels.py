"""Torch-tensor front end over the C-ABI kernels (device memory is owned by torch).

Each function validates shapes/dtypes/devices, then calls exactly one
`zb_*` entry point on the current CUDA stream.  Nothing here computes on the
CPU: a missing library or a non-CUDA tensor raises.
"""

from __future__ import annotations

import torch

from ._lib import call as _call

# Device kernel launches issued per C-ABI entry point (for the bench's gpu_launches).
_LAUNCHES_PER_CALL = {"zb_attn_bwd": 3, "zb_layernorm_bwd": 2,
                      "zb_layernorm_bwd_ex": 2, "zb_rmsnorm_bwd": 2}
_launches = [0]


def call(name, *args):
    _call(name, *args)
    _launches[0] += _LAUNCHES_PER_CALL.get(name, 1)


def reset_launch_count():
    _launches[0] = 0


def launch_count():
    return _launches[0]

# GEMM epilogues (csrc/gemm_sm100.cu)
EPI_BF16 = 0
EPI_BIAS = 1
EPI_BIAS_GELU = 2
EPI_BIAS_RESID = 3
EPI_GELU_BWD = 4
EPI_F32 = 5
EPI_RESID = 6
EPI_BIAS_GELU_NA = 7   # C = gelu(acc + bias), no pre-activation output (forward pass)


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libzorse_b200 kernels take CUDA tensors only (no CPU fallback)")


def _gemm_args(a, b, out, a_t, b_t, bias, resid, aux, M, N, K):
    _need_cuda(a, b, out, bias, resid, aux)
    if a_t:
        K_, M_ = a.shape
    else:
        M_, K_ = a.shape
    if b_t:
        K2, N_ = b.shape
    else:
        N_, K2 = b.shape
    if K_ != K2:
        raise ValueError(f"gemm: K mismatch {tuple(a.shape)} {tuple(b.shape)}")
    M = M_ if M is None else M
    N = N_ if N is None else N
    K = K_ if K is None else K
    for t in (a, b, out):
        if t.stride(-1) != 1:
            raise ValueError("gemm operands need unit inner stride")
    return (M, N, K, a.stride(0), b.stride(0), out.stride(0),
            resid.stride(0) if resid is not None else 0, aux.stride(0) if aux is not None else 0,
            int(a_t), int(b_t))


def gemm(a, b, out, *, a_t=False, b_t=False, epilogue=EPI_BF16, bias=None, resid=None,
         aux=None, beta=0.0, M=None, N=None, K=None):
    """out[M,N] = op(a) @ op(b)^T with tcgen05.

    a: [M,K] (a_t=False) or [K,M] (a_t=True);  b: [N,K] (b_t=False) or [K,N] (b_t=True).
    All 2-D, row-major with unit inner stride; leading dims taken from stride(0).
    The tile comes from the committed B200 tile table, else the cost model.
    """
    dims = _gemm_args(a, b, out, a_t, b_t, bias, resid, aux, M, N, K)
    call("zb_gemm_bf16", _ptr(a), _ptr(b), _ptr(out), _ptr(bias), _ptr(resid), _ptr(aux),
         *dims, epilogue, float(beta), _stream())
    return out


def gemm_tile(a, b, out, *, pair=-1, bn=0, splits=0, raster=-1, tma_epi=True, a_t=False,
              b_t=False, epilogue=EPI_BF16, bias=None, resid=None, aux=None, beta=0.0):
    """``gemm`` with an explicit tile (tests / tuning / benchmarks): pair 0 = 1-CTA,
    1 = CTA pair, 2 = multicast pairs; bn 128/192/256; K splits (fp32 beta=1 only);
    raster 0 = M-fastest, 1 = N-fastest; tma_epi False = direct-store epilogue.
    Negative / zero values keep the cost model's pick for that field."""
    dims = _gemm_args(a, b, out, a_t, b_t, bias, resid, aux, None, None, None)
    call("zb_gemm_bf16_tile", _ptr(a), _ptr(b), _ptr(out), _ptr(bias), _ptr(resid), _ptr(aux),
         *dims, epilogue, float(beta), int(pair), int(bn), int(splits), int(raster),
         int(bool(tma_epi)), _stream())
    return out


def gemm_choice(M, N, K, *, a_t=False, b_t=False, epilogue=EPI_BF16, beta=0.0, ldc=None):
    """(pair, bn, splits, from_table) that ``gemm`` uses for this shape."""
    import ctypes
    outs = [ctypes.c_int() for _ in range(4)]
    call("zb_gemm_choice", M, N, K, int(a_t), int(b_t), epilogue, float(beta),
         N if ldc is None else ldc, *[ctypes.byref(o) for o in outs])
    return tuple(o.value for o in outs[:3]) + (bool(outs[3].value),)


def gemm_tune(a, b, out, *, a_t=False, b_t=False, epilogue=EPI_BF16, bias=None, resid=None,
              aux=None, beta=0.0):
    """Measure the candidate tiles for this call's shape (synchronises; never inside
    graph capture) and return the fastest (pair, bn, splits).  scripts/tune_gemm.py
    writes the results into the committed tile table."""
    import ctypes
    dims = _gemm_args(a, b, out, a_t, b_t, bias, resid, aux, None, None, None)
    outs = [ctypes.c_int() for _ in range(3)]
    call("zb_gemm_tune", _ptr(a), _ptr(b), _ptr(bias), _ptr(resid), _ptr(aux), *dims, epilogue,
         float(beta), *[ctypes.byref(o) for o in outs], _stream())
    return tuple(o.value for o in outs)


def layernorm_fwd(x, w, b, y, mean, rstd, eps=1e-5):
    _need_cuda(x, w, b, y, mean, rstd)
    rows, d = x.shape
    call("zb_layernorm_fwd", _ptr(x), _ptr(w), _ptr(b), _ptr(y), _ptr(mean), _ptr(rstd),
         None, rows, d, float(eps), _stream())


def layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=None, db_accum=None, db_out=None,
                  phase=0):
    """dx (+)= LN'(dy); dw, db (fp32) += parameter grads.  dx_accum: residual grad to add.
    db_accum / db_out (fp32, optional, together): += column sums of dx_accum / of dx.
    phase 1 / 2: only the dx launch / only the (dw, db, db_accum, db_out) column pass."""
    _need_cuda(dy, x, w, mean, rstd, dx, dw, db, dx_accum, db_accum, db_out)
    rows, d = x.shape
    if phase:
        call("zb_layernorm_bwd_phase", _ptr(dy), _ptr(x), _ptr(w), _ptr(mean), _ptr(rstd),
             _ptr(dx), _ptr(dw), _ptr(db), _ptr(dx_accum), _ptr(db_accum), _ptr(db_out), rows, d,
             int(phase), _stream())
        return
    if db_accum is not None or db_out is not None:
        call("zb_layernorm_bwd_ex", _ptr(dy), _ptr(x), _ptr(w), _ptr(mean), _ptr(rstd), _ptr(dx),
             _ptr(dw), _ptr(db), _ptr(dx_accum), _ptr(db_accum), _ptr(db_out), rows, d,
             _stream())
        return
    call("zb_layernorm_bwd", _ptr(dy), _ptr(x), _ptr(w), _ptr(mean), _ptr(rstd), _ptr(dx),
         _ptr(dw), _ptr(db), _ptr(dx_accum), rows, d, _stream())


def embedding_fwd(tokens, wte, wpe, out, seq_len):
    _need_cuda(tokens, wte, wpe, out)
    rows, d = out.shape
    call("zb_embedding_fwd", _ptr(tokens), _ptr(wte), _ptr(wpe), _ptr(out), rows, d, seq_len,
         _stream())


def embedding_bwd(tokens, dout, dwte, dwpe, seq_len):
    _need_cuda(tokens, dout, dwte, dwpe)
    rows, d = dout.shape
    call("zb_embedding_bwd", _ptr(tokens), _ptr(dout), _ptr(dwte), _ptr(dwpe), rows, d, seq_len,
         _stream())


def xent_fwd_bwd(logits, labels, loss_sum, dlogits, scale):
    """Per-row softmax cross-entropy: loss_sum (+)= sum_rows CE; dlogits = (p - 1hot) * scale."""
    _need_cuda(logits, labels, loss_sum, dlogits)
    rows, V = logits.shape
    call("zb_xent_fwd_bwd", _ptr(logits), _ptr(labels), _ptr(loss_sum), _ptr(dlogits), rows, V,
         logits.stride(0), float(scale), _stream())


def bias_grad(dy, db):
    """db (fp32) += column sums of dy [rows, n] (bf16)."""
    _need_cuda(dy, db)
    rows, n = dy.shape
    call("zb_bias_grad", _ptr(dy), _ptr(db), rows, n, dy.stride(0), _stream())


def attn_fwd(qkv, out, lse, n_seq, seq_len, n_head, head_dim, scale):
    """Causal attention forward on tcgen05/TMEM (csrc/attn_sm100.cu)."""
    _need_cuda(qkv, out, lse)
    call("zb_attn_fwd", _ptr(qkv), _ptr(out), _ptr(lse), n_seq, seq_len, n_head, head_dim,
         qkv.stride(0), float(scale), _stream())


def attn_bwd(qkv, out, dout, lse, dqkv, dq_accum, delta, n_seq, seq_len, n_head, head_dim,
             scale):
    """Causal attention backward on tcgen05/TMEM (csrc/attn_bwd_sm100.cu)."""
    _need_cuda(qkv, out, dout, lse, dqkv, dq_accum, delta)
    call("zb_attn_bwd", _ptr(qkv), _ptr(out), _ptr(dout), _ptr(lse), _ptr(dqkv), _ptr(dq_accum),
         _ptr(delta), n_seq, seq_len, n_head, head_dim, qkv.stride(0), float(scale), _stream())


def adamw_shard(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, lr, beta1, beta2, eps,
                weight_decay, grad_scale, step):
    """step: python int, or an int32 CUDA tensor holding t (read on the device)."""
    _need_cuda(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq)
    n = master.numel()
    if isinstance(step, torch.Tensor):
        _need_cuda(step)
        call("zb_adamw_shard_dstep", _ptr(master), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad),
             _ptr(param_bf16), _ptr(sumsq), n, float(lr), float(beta1), float(beta2), float(eps),
             float(weight_decay), float(grad_scale), _ptr(step), _stream())
        return
    call("zb_adamw_shard", _ptr(master), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad),
         _ptr(param_bf16), _ptr(sumsq), n, float(lr), float(beta1), float(beta2), float(eps),
         float(weight_decay), float(grad_scale), int(step), _stream())


def embed_mark(tokens, rows, mark, step_dev):
    """mark[tok] = step (device counter) for every token (row-split embedding update)."""
    _need_cuda(tokens, mark, step_dev)
    call("zb_embed_mark", _ptr(tokens), tokens.numel(), int(rows), _ptr(mark), _ptr(step_dev),
         _stream())


def embed_zero_rows(tokens, grad_table):
    """grad_table[tok, :] = 0 for every token; grad_table: fp32 [rows, d]."""
    _need_cuda(tokens, grad_table)
    rows, d = grad_table.shape
    call("zb_embed_zero_rows", _ptr(tokens), tokens.numel(), rows, _ptr(grad_table), d, _stream())


def adamw_rows(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, mark, marked, lr, beta1,
               beta2, eps, weight_decay, grad_scale, step_dev):
    """AdamW over the rows r of [rows, d] tables with (mark[r] == step) == marked;
    marked=False: g = 0, ``grad`` unused (may be None)."""
    _need_cuda(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, mark, step_dev)
    rows, d = master.shape
    call("zb_adamw_rows_dstep", _ptr(master), _ptr(exp_avg), _ptr(exp_avg_sq), _ptr(grad),
         _ptr(param_bf16), _ptr(sumsq), rows, d, _ptr(mark), int(bool(marked)), float(lr),
         float(beta1), float(beta2), float(eps), float(weight_decay), float(grad_scale),
         _ptr(step_dev), _stream())


def cast_f32_bf16(src, dst):
    _need_cuda(src, dst)
    call("zb_cast_f32_bf16", _ptr(src), _ptr(dst), src.numel(), _stream())


def fill_f32(t, value):
    _need_cuda(t)
    call("zb_fill_f32", _ptr(t), float(value), t.numel(), _stream())


def add_bf16(a, b, out):
    _need_cuda(a, b, out)
    call("zb_add_bf16", _ptr(a), _ptr(b), _ptr(out), a.numel(), _stream())


def step_increment(step_dev):
    """step_dev (int32 CUDA tensor) += 1 on the device."""
    _need_cuda(step_dev)
    call("zb_step_increment", _ptr(step_dev), _stream())


def rmsnorm_fwd(x, w, y, rstd, eps=1e-5):
    _need_cuda(x, w, y, rstd)
    rows, d = x.shape
    call("zb_rmsnorm_fwd", _ptr(x), _ptr(w), _ptr(y), _ptr(rstd), rows, d, float(eps), _stream())


def rmsnorm_bwd(dy, x, w, rstd, dx, dw, dx_accum=None):
    _need_cuda(dy, x, w, rstd, dx, dw, dx_accum)
    rows, d = x.shape
    call("zb_rmsnorm_bwd", _ptr(dy), _ptr(x), _ptr(w), _ptr(rstd), _ptr(dx), _ptr(dw),
         _ptr(dx_accum), rows, d, _stream())


def rope(qkv, seq_len, n_head, head_dim, theta=10000.0, inverse=False):
    _need_cuda(qkv)
    call("zb_rope", _ptr(qkv), qkv.shape[0], seq_len, n_head, head_dim, qkv.stride(0),
         float(theta), int(inverse), _stream())


def swiglu_fwd(gu, out):
    _need_cuda(gu, out)
    call("zb_swiglu_fwd", _ptr(gu), _ptr(out), out.shape[0], out.shape[1], _stream())


def swiglu_bwd(gu, dout, dgu):
    _need_cuda(gu, dout, dgu)
    call("zb_swiglu_bwd", _ptr(gu), _ptr(dout), _ptr(dgu), dout.shape[0], dout.shape[1], _stream())
