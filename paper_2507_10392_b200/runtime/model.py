"""GPT transformer block / embedding / head expressed as kernel calls.

A layer's parameters live in ONE flat buffer (bf16 for compute, fp32 for the
master copy, fp32 for gradients) so that the uneven ZeRO-3 AllGather-v /
ReduceScatter-v of a layer is a single in-place collective on contiguous
memory.  Flat order per layer (12 d^2 + 13 d elements when f = 4d, the
reference's ``transformer_params_per_layer`` fixtures.py:176-178):

    ln1_w[d] ln1_b[d] qkv_w[3d,d] qkv_b[3d] proj_w[d,d] proj_b[d]
    ln2_w[d] ln2_b[d] fc1_w[f,d] fc1_b[f] fc2_w[d,f] fc2_b[d]

Embedding (first global stage) and head (last global stage) are not planner
layers (the reference assumes the first/last stages carry them,
configure.py:354-356); they get their own flat buffers:

    embed: wte[V,d] wpe[S,d]          head: lnf_w[d] lnf_b[d] head_w[V,d]

Every op is a call into ``ops`` (``paper_2507_10392_b200.kernels`` on B200).
Activation layout: token-major [tokens, d] bf16; a microbatch slice of
``n`` sequences is n*S contiguous rows.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch

from ..plan.emulated import ModelConfig

EPI_BF16, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_GELU_BWD, EPI_F32, EPI_RESID, EPI_BIAS_GELU_NA = range(8)


class FlatLayout:
    """Named tensor views into a flat buffer."""

    def __init__(self, entries: List[Tuple[str, Tuple[int, ...]]]):
        self.entries = []
        off = 0
        for name, shape in entries:
            n = 1
            for s in shape:
                n *= s
            self.entries.append((name, off, shape))
            off += n
        self.numel = off

    def views(self, flat: torch.Tensor) -> Dict[str, torch.Tensor]:
        if flat.numel() != self.numel:
            raise ValueError(f"flat buffer has {flat.numel()} elements, layout needs {self.numel}")
        out = {}
        for name, off, shape in self.entries:
            n = 1
            for s in shape:
                n *= s
            out[name] = flat[off:off + n].view(*shape)
        return out


def layer_layout(cfg: ModelConfig) -> FlatLayout:
    d, f = cfg.d_model, cfg.ffn
    if cfg.family == "llama":
        # 4d^2 + 3df + 2d (SURVEY §8 notation); gate and up projections fused [2f, d]
        return FlatLayout([("attn_norm", (d,)), ("qkv_w", (3 * d, d)), ("o_w", (d, d)),
                           ("mlp_norm", (d,)), ("gu_w", (2 * f, d)), ("down_w", (d, f))])
    return FlatLayout([("ln1_w", (d,)), ("ln1_b", (d,)), ("qkv_w", (3 * d, d)), ("qkv_b", (3 * d,)),
                       ("proj_w", (d, d)), ("proj_b", (d,)), ("ln2_w", (d,)), ("ln2_b", (d,)),
                       ("fc1_w", (f, d)), ("fc1_b", (f,)), ("fc2_w", (d, f)), ("fc2_b", (d,))])


def embed_layout(cfg: ModelConfig) -> FlatLayout:
    if cfg.family == "llama":
        return FlatLayout([("wte", (cfg.vocab, cfg.d_model))])
    return FlatLayout([("wte", (cfg.vocab, cfg.d_model)), ("wpe", (cfg.seq_len, cfg.d_model))])


def head_layout(cfg: ModelConfig) -> FlatLayout:
    d = cfg.d_model
    if cfg.family == "llama":
        return FlatLayout([("norm_w", (d,)), ("head_w", (cfg.vocab, d))])
    return FlatLayout([("lnf_w", (d,)), ("lnf_b", (d,)), ("head_w", (cfg.vocab, d))])


def init_flat(layout: FlatLayout, kind: str, index: int, cfg: ModelConfig, seed: int,
              device="cpu") -> torch.Tensor:
    """Deterministic fp32 init of one flat buffer (GPT-2 scheme): N(0, 0.02)
    weights, residual projections N(0, 0.02/sqrt(2L)), LayerNorm w=1 b=0,
    biases 0.  Each tensor draws from its own generator so any rank can build
    any buffer independently."""
    flat = torch.empty(layout.numel, dtype=torch.float32, device=device)
    views = layout.views(flat)
    resid_std = 0.02 / math.sqrt(2 * cfg.n_layer)
    for t_idx, (name, _, shape) in enumerate(layout.entries):
        v = views[name]
        if name.endswith("_b"):
            v.zero_()
        elif name.startswith("ln") or name.endswith("norm") or name == "norm_w":
            v.fill_(1.0)
        else:
            std = resid_std if name in ("proj_w", "fc2_w") else 0.02
            g = torch.Generator(device=device)
            g.manual_seed(seed * 1_000_003 + {"layer": 0, "embed": 1, "head": 2}[kind] * 100_003
                          + index * 101 + t_idx)
            v.normal_(0.0, std, generator=g)
    return flat


@dataclass
class LayerActs:
    """Per-layer activations kept between Recompute and Bwd of one microbatch."""

    h1: torch.Tensor      # LN1(x)            [n, d]
    mean1: torch.Tensor
    rstd1: torch.Tensor
    qkv: torch.Tensor     # [n, 3d]
    attn: torch.Tensor    # [n, d]
    lse: torch.Tensor     # [seqs, H, S]
    x_mid: torch.Tensor   # x + proj(attn)   [n, d]
    h2: torch.Tensor      # LN2(x_mid)
    mean2: torch.Tensor
    rstd2: torch.Tensor
    u: torch.Tensor       # fc1 pre-activation [n, f]
    g: torch.Tensor       # gelu(u)            [n, f]


@dataclass
class LlamaActs:
    h1: torch.Tensor      # RMSNorm1(x)       [n, d]
    rstd1: torch.Tensor
    qkv: torch.Tensor     # post-RoPE q,k | v  [n, 3d]
    attn: torch.Tensor    # [n, d]
    lse: torch.Tensor
    x_mid: torch.Tensor   # [n, d]
    h2: torch.Tensor      # RMSNorm2(x_mid)
    rstd2: torch.Tensor
    gu: torch.Tensor      # [gate | up]       [n, 2f]
    m: torch.Tensor       # silu(gate) * up   [n, f]


def alloc_acts(cfg: ModelConfig, n_tok: int, device):
    if cfg.family == "llama":
        d, f, H, S = cfg.d_model, cfg.ffn, cfg.n_head, cfg.seq_len
        n = max(n_tok, 1)
        bf = dict(device=device, dtype=torch.bfloat16)
        return LlamaActs(h1=torch.empty(n, d, **bf), rstd1=torch.empty(n, device=device),
                         qkv=torch.empty(n, 3 * d, **bf), attn=torch.empty(n, d, **bf),
                         lse=torch.empty(max(n_tok // S, 1), H, S, device=device),
                         x_mid=torch.empty(n, d, **bf), h2=torch.empty(n, d, **bf),
                         rstd2=torch.empty(n, device=device), gu=torch.empty(n, 2 * f, **bf),
                         m=torch.empty(n, f, **bf))
    return _alloc_gpt_acts(cfg, n_tok, device)


def _alloc_gpt_acts(cfg: ModelConfig, n_tok: int, device) -> LayerActs:
    d, f, H, S = cfg.d_model, cfg.ffn, cfg.n_head, cfg.seq_len
    seqs = max(n_tok // S, 1)
    bf = dict(device=device, dtype=torch.bfloat16)
    fp = dict(device=device, dtype=torch.float32)
    n = max(n_tok, 1)
    return LayerActs(h1=torch.empty(n, d, **bf), mean1=torch.empty(n, **fp), rstd1=torch.empty(n, **fp),
                     qkv=torch.empty(n, 3 * d, **bf), attn=torch.empty(n, d, **bf),
                     lse=torch.empty(seqs, H, S, **fp), x_mid=torch.empty(n, d, **bf),
                     h2=torch.empty(n, d, **bf), mean2=torch.empty(n, **fp), rstd2=torch.empty(n, **fp),
                     u=torch.empty(n, f, **bf), g=torch.empty(n, f, **bf))


@dataclass
class BwdScratch:
    dh: torch.Tensor      # [n, d]
    dx_mid: torch.Tensor  # [n, d]
    da: torch.Tensor      # [n, d]
    dqkv: torch.Tensor    # [n, 3d]
    delta: torch.Tensor   # [seqs, H, S]
    dq_accum: Optional[torch.Tensor] = None  # [n, d] fp32: fused attention backward (D = 64)


def alloc_bwd_scratch(cfg: ModelConfig, n_tok: int, device) -> BwdScratch:
    d, H, S = cfg.d_model, cfg.n_head, cfg.seq_len
    n = max(n_tok, 1)
    bf = dict(device=device, dtype=torch.bfloat16)
    return BwdScratch(dh=torch.empty(n, d, **bf), dx_mid=torch.empty(n, d, **bf),
                      da=torch.empty(n, d, **bf), dqkv=torch.empty(n, 3 * d, **bf),
                      delta=torch.empty(max(n_tok // S, 1), H, S, device=device),
                      dq_accum=(torch.empty(n, d, device=device, dtype=torch.float32)
                                if cfg.head_dim == 64 else None))


class WgradLane:
    """Weight-gradient GEMMs of a block backward on a second CUDA stream.

    In a linear layer's backward only the data gradient (dgrad) is on the critical
    path; the weight gradient (wgrad) is read by nothing until the ministage's
    ReduceScatter / optimizer.  Forking each wgrad off the compute stream (after the
    producer of its operands) lets its CTAs fill the SMs the dgrad chain leaves idle
    (wave tails, small HBM-bound kernels).  ``join`` at the end of the block makes
    the compute stream wait for every forked GEMM before the block's buffers are
    reused (the next block's recompute overwrites them).  CPU tensors (tests' torch
    twin) run everything inline; ``enabled = False`` serialises the lane (the bench's
    per-launch GEMM timing)."""

    def __init__(self):
        self.stream = None
        self.pending = False
        self.enabled = True

    def fork(self, t: torch.Tensor):
        """Context for one wgrad launch, ordered after the compute stream's work so far."""
        if not (self.enabled and t.is_cuda):
            return _Inline()
        if self.stream is None:
            self.stream = torch.cuda.Stream(device=t.device)
        main = torch.cuda.current_stream(t.device)
        self.stream.wait_stream(main)
        self.pending = True
        return torch.cuda.stream(self.stream)

    def join(self, t: torch.Tensor) -> None:
        if self.pending:
            torch.cuda.current_stream(t.device).wait_stream(self.stream)
            self.pending = False


class _Inline:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class GptOps:
    """Composes one rank's transformer math out of kernel calls."""

    def __init__(self, cfg: ModelConfig, ops):
        if cfg.family != "gpt":
            raise NotImplementedError(f"model family {cfg.family!r} is not wired yet")
        self.cfg, self.ops = cfg, ops
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        self.wlane = WgradLane()

    def layer_fwd(self, p: Dict[str, torch.Tensor], x: torch.Tensor, out: torch.Tensor,
                  a: LayerActs, n_tok: int, need_out: bool = True, kept=False,
                  keep_preact=False) -> None:
        """out = block(x); fills ``a`` (the recompute set).  ``need_out=False``
        (activation recompute) skips the fc2 GEMM: backward never reads the
        block output, only its internals.  ``kept``: a.attn / a.lse / a.x_mid hold
        the attention block's outputs of this (layer, microbatch) kept from the
        forward pass, so the recompute skips the attention forward and the
        projection GEMM (selective recompute).  ``keep_preact``: the forward also
        writes the fc1 pre-activation (the backward reads it when nothing is
        recomputed)."""
        o, cfg = self.ops, self.cfg
        n_seq = n_tok // cfg.seq_len
        o.layernorm_fwd(x, p["ln1_w"], p["ln1_b"], a.h1[:n_tok], a.mean1[:n_tok], a.rstd1[:n_tok])
        o.gemm(a.h1[:n_tok], p["qkv_w"], a.qkv[:n_tok], epilogue=EPI_BIAS, bias=p["qkv_b"])
        if not kept:
            o.attn_fwd(a.qkv[:n_tok], a.attn[:n_tok], a.lse[:n_seq], n_seq, cfg.seq_len,
                       cfg.n_head, cfg.head_dim, self.scale)
            o.gemm(a.attn[:n_tok], p["proj_w"], a.x_mid[:n_tok], epilogue=EPI_BIAS_RESID,
                   bias=p["proj_b"], resid=x)
        o.layernorm_fwd(a.x_mid[:n_tok], p["ln2_w"], p["ln2_b"], a.h2[:n_tok], a.mean2[:n_tok],
                        a.rstd2[:n_tok])
        if need_out and not keep_preact:  # backward reads the recompute's pre-activation
            o.gemm(a.h2[:n_tok], p["fc1_w"], a.g[:n_tok], epilogue=EPI_BIAS_GELU_NA,
                   bias=p["fc1_b"])
        else:
            o.gemm(a.h2[:n_tok], p["fc1_w"], a.g[:n_tok], epilogue=EPI_BIAS_GELU, bias=p["fc1_b"],
                   aux=a.u[:n_tok])
        if need_out:
            o.gemm(a.g[:n_tok], p["fc2_w"], out, epilogue=EPI_BIAS_RESID, bias=p["fc2_b"],
                   resid=a.x_mid[:n_tok])

    def layer_bwd(self, p: Dict[str, torch.Tensor], gr: Dict[str, torch.Tensor], x: torch.Tensor,
                  dy: torch.Tensor, dx: torch.Tensor, a: LayerActs, s: BwdScratch,
                  n_tok: int) -> None:
        """dx = d(block)/dx . dy ; parameter grads accumulate into ``gr`` (fp32).
        (The weight-gradient GEMMs always accumulate: their tiles split K and reduce-add
        into the slot, which therefore has to start at zero.)"""
        o, cfg = self.ops, self.cfg
        n_seq = n_tok // cfg.seq_len
        n = n_tok
        w = self.wlane  # weight grads off the critical path (operands are not rewritten
        #                  before the join at the end of the block)
        # MLP: out = x_mid + g W2^T + b2
        with w.fork(dy):
            o.gemm(dy, a.g[:n], gr["fc2_w"], a_t=True, b_t=True, epilogue=EPI_F32, beta=1.0)
        # fc2 / proj bias grads: column sums of dy / dx_mid, folded into LN2's backward
        o.gemm(dy, p["fc2_w"], a.u[:n], b_t=True, epilogue=EPI_GELU_BWD, aux=a.u[:n])  # du (in place)
        with w.fork(dy):
            o.gemm(a.u[:n], a.h2[:n], gr["fc1_w"], a_t=True, b_t=True, epilogue=EPI_F32, beta=1.0)
            o.bias_grad(a.u[:n], gr["fc1_b"])
        o.gemm(a.u[:n], p["fc1_w"], s.dh[:n], b_t=True)
        o.layernorm_bwd(s.dh[:n], a.x_mid[:n], p["ln2_w"], a.mean2[:n], a.rstd2[:n], s.dx_mid[:n],
                        gr["ln2_w"], gr["ln2_b"], dx_accum=dy, db_accum=gr["fc2_b"],
                        db_out=gr["proj_b"])
        # attention: x_mid = x + attn W_o^T + b_o
        with w.fork(dy):
            o.gemm(s.dx_mid[:n], a.attn[:n], gr["proj_w"], a_t=True, b_t=True, epilogue=EPI_F32,
                   beta=1.0)
        o.gemm(s.dx_mid[:n], p["proj_w"], s.da[:n], b_t=True)
        o.attn_bwd(a.qkv[:n], a.attn[:n], s.da[:n], a.lse[:n_seq], s.dqkv[:n],
                   s.dq_accum[:n] if s.dq_accum is not None else None,
                   s.delta[:n_seq], n_seq, cfg.seq_len, cfg.n_head, cfg.head_dim, self.scale)
        with w.fork(dy):
            o.gemm(s.dqkv[:n], a.h1[:n], gr["qkv_w"], a_t=True, b_t=True, epilogue=EPI_F32,
                   beta=1.0)
            o.bias_grad(s.dqkv[:n], gr["qkv_b"])
        o.gemm(s.dqkv[:n], p["qkv_w"], s.dh[:n], b_t=True)
        o.layernorm_bwd(s.dh[:n], x, p["ln1_w"], a.mean1[:n], a.rstd1[:n], dx, gr["ln1_w"],
                        gr["ln1_b"], dx_accum=s.dx_mid[:n])
        w.join(dy)

    def embed_fwd(self, p, tokens, out, n_tok):
        self.ops.embedding_fwd(tokens[:n_tok], p["wte"], p["wpe"], out, self.cfg.seq_len)

    def embed_bwd(self, gr, tokens, dx, n_tok):
        self.ops.embedding_bwd(tokens[:n_tok], dx, gr["wte"], gr["wpe"], self.cfg.seq_len)

    def head_fwd_bwd(self, p, gr, x, labels, dx, logits, hf, mean, rstd, dhf, loss_sum, scale,
                     n_tok, dhf32=None, first=False):
        """Final LayerNorm + LM head + cross-entropy, and straight away its
        backward: dx (grad of the last block's output) and head grads."""
        o = self.ops
        n = n_tok
        o.layernorm_fwd(x, p["lnf_w"], p["lnf_b"], hf[:n], mean[:n], rstd[:n])
        o.gemm(hf[:n], p["head_w"], logits[:n])
        o.xent_fwd_bwd(logits[:n], labels[:n], loss_sum, logits[:n], scale)
        # (LM-head wgrad inline: forking it measured neutral; both GEMMs fill the GPU).
        # first: the first accumulation into a freshly bound gradient slot overwrites
        # (beta = 0; its tiles do not split K), so the slot's head_w span is not cleared.
        o.gemm(logits[:n], hf[:n], gr["head_w"], a_t=True, b_t=True, epilogue=EPI_F32,
               beta=0.0 if first else 1.0)
        head_dgrad(o, logits[:n], p["head_w"], dhf[:n], None if dhf32 is None else dhf32[:n])
        o.layernorm_bwd(dhf[:n], x, p["lnf_w"], mean[:n], rstd[:n], dx, gr["lnf_w"], gr["lnf_b"])


class LlamaOps:
    """Llama block (pre-RMSNorm, RoPE, SwiGLU, no biases) as kernel calls; same
    interface as GptOps."""

    ROPE_THETA = 10000.0

    def __init__(self, cfg: ModelConfig, ops):
        self.cfg, self.ops = cfg, ops
        self.scale = 1.0 / math.sqrt(cfg.head_dim)
        self.wlane = WgradLane()

    def layer_fwd(self, p, x, out, a: LlamaActs, n_tok: int, need_out: bool = True,
                  kept=False, keep_preact=False) -> None:
        o, cfg = self.ops, self.cfg
        n = n_tok
        n_seq = n // cfg.seq_len
        o.rmsnorm_fwd(x, p["attn_norm"], a.h1[:n], a.rstd1[:n])
        o.gemm(a.h1[:n], p["qkv_w"], a.qkv[:n])
        o.rope(a.qkv[:n], cfg.seq_len, cfg.n_head, cfg.head_dim, self.ROPE_THETA)
        if not kept:
            o.attn_fwd(a.qkv[:n], a.attn[:n], a.lse[:n_seq], n_seq, cfg.seq_len, cfg.n_head,
                       cfg.head_dim, self.scale)
            o.gemm(a.attn[:n], p["o_w"], a.x_mid[:n], epilogue=EPI_RESID, resid=x)
        o.rmsnorm_fwd(a.x_mid[:n], p["mlp_norm"], a.h2[:n], a.rstd2[:n])
        o.gemm(a.h2[:n], p["gu_w"], a.gu[:n])
        o.swiglu_fwd(a.gu[:n], a.m[:n])
        if need_out:
            o.gemm(a.m[:n], p["down_w"], out, epilogue=EPI_RESID, resid=a.x_mid[:n])

    def layer_bwd(self, p, gr, x, dy, dx, a: LlamaActs, s: BwdScratch, n_tok: int) -> None:
        o, cfg = self.ops, self.cfg
        n = n_tok
        n_seq = n // cfg.seq_len
        w = self.wlane  # see GptOps.layer_bwd
        # down-proj wgrad stays inline: its dgrad overwrites the operand m in place
        o.gemm(dy, a.m[:n], gr["down_w"], a_t=True, b_t=True, epilogue=EPI_F32, beta=1.0)
        o.gemm(dy, p["down_w"], a.m[:n], b_t=True)                 # dm (m no longer needed)
        o.swiglu_bwd(a.gu[:n], a.m[:n], a.gu[:n])                  # d[gate|up] in place
        with w.fork(dy):
            o.gemm(a.gu[:n], a.h2[:n], gr["gu_w"], a_t=True, b_t=True, epilogue=EPI_F32, beta=1.0)
        o.gemm(a.gu[:n], p["gu_w"], s.dh[:n], b_t=True)
        o.rmsnorm_bwd(s.dh[:n], a.x_mid[:n], p["mlp_norm"], a.rstd2[:n], s.dx_mid[:n],
                      gr["mlp_norm"], dx_accum=dy)
        with w.fork(dy):
            o.gemm(s.dx_mid[:n], a.attn[:n], gr["o_w"], a_t=True, b_t=True, epilogue=EPI_F32,
                   beta=1.0)
        o.gemm(s.dx_mid[:n], p["o_w"], s.da[:n], b_t=True)
        o.attn_bwd(a.qkv[:n], a.attn[:n], s.da[:n], a.lse[:n_seq], s.dqkv[:n],
                   s.dq_accum[:n] if s.dq_accum is not None else None,
                   s.delta[:n_seq], n_seq, cfg.seq_len, cfg.n_head, cfg.head_dim, self.scale)
        o.rope(s.dqkv[:n], cfg.seq_len, cfg.n_head, cfg.head_dim, self.ROPE_THETA, inverse=True)
        with w.fork(dy):
            o.gemm(s.dqkv[:n], a.h1[:n], gr["qkv_w"], a_t=True, b_t=True, epilogue=EPI_F32,
                   beta=1.0)
        o.gemm(s.dqkv[:n], p["qkv_w"], s.dh[:n], b_t=True)
        o.rmsnorm_bwd(s.dh[:n], x, p["attn_norm"], a.rstd1[:n], dx, gr["attn_norm"],
                      dx_accum=s.dx_mid[:n])
        w.join(dy)

    def embed_fwd(self, p, tokens, out, n_tok):
        self.ops.embedding_fwd(tokens[:n_tok], p["wte"], None, out, self.cfg.seq_len)

    def embed_bwd(self, gr, tokens, dx, n_tok):
        self.ops.embedding_bwd(tokens[:n_tok], dx, gr["wte"], None, self.cfg.seq_len)

    def head_fwd_bwd(self, p, gr, x, labels, dx, logits, hf, mean, rstd, dhf, loss_sum, scale,
                     n_tok, dhf32=None, first=False):
        o = self.ops
        n = n_tok
        o.rmsnorm_fwd(x, p["norm_w"], hf[:n], rstd[:n])
        o.gemm(hf[:n], p["head_w"], logits[:n])
        o.xent_fwd_bwd(logits[:n], labels[:n], loss_sum, logits[:n], scale)
        # (LM-head wgrad inline: forking it measured neutral; both GEMMs fill the GPU).
        # first: the first accumulation into a freshly bound gradient slot overwrites
        # (beta = 0; its tiles do not split K), so the slot's head_w span is not cleared.
        o.gemm(logits[:n], hf[:n], gr["head_w"], a_t=True, b_t=True, epilogue=EPI_F32,
               beta=0.0 if first else 1.0)
        head_dgrad(o, logits[:n], p["head_w"], dhf[:n], None if dhf32 is None else dhf32[:n])
        o.rmsnorm_bwd(dhf[:n], x, p["norm_w"], rstd[:n], dx, gr["norm_w"])


def head_dgrad(o, dlogits, head_w, dhf, dhf32=None) -> None:
    """dhf = dlogits @ head_w.  The output has only d columns (3-4 tiles across) and K is
    the vocabulary, so a bf16 GEMM runs 1.3 waves of tiles; accumulating in fp32 with
    K split (TMA reduce-add) fills the GPU and the cast back is a 6 us pass: 529 -> 467
    us at GPT-2 small (profiles/r02_gemm_ab.jsonl)."""
    if dhf32 is None:
        o.gemm(dlogits, head_w, dhf, b_t=True)
        return
    o.fill_f32(dhf32, 0.0)
    o.gemm(dlogits, head_w, dhf32, b_t=True, epilogue=EPI_F32, beta=1.0)
    o.cast_f32_bf16(dhf32, dhf)


def make_model_ops(cfg: ModelConfig, ops):
    if cfg.family == "gpt":
        return GptOps(cfg, ops)
    if cfg.family == "llama":
        return LlamaOps(cfg, ops)
    raise NotImplementedError(f"model family {cfg.family!r}")
