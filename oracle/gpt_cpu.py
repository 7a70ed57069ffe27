"""TEST INFRASTRUCTURE ONLY — fp32 CPU oracle for one GPT training step.

Semantics (the contract the B200 executor implements, whatever the plan):
  x = wte[tok] + wpe[pos];  per block (pre-LN):
      x = x + proj(causal_attn(qkv(LN1(x))));  x = x + fc2(gelu_tanh(fc1(LN2(x))))
  logits = LNf(x) @ head_w^T;  loss = sum CE / (global_batch * seq_len)
  AdamW (torch.optim.AdamW rule, decoupled decay on every parameter).
The plan only changes WHERE and in WHICH ORDER this runs (shares, stages,
ministage-interleaved optimizer after the last backward of each ministage);
since every forward of an iteration precedes every optimizer update of the
parameters it reads, the math equals this full-batch step.
"""

from __future__ import annotations

import math
from typing import Dict

import torch
import torch.nn.functional as F

from paper_2507_10392_b200.plan.emulated import ModelConfig
from paper_2507_10392_b200.runtime.model import (embed_layout, head_layout, init_flat,
                                                 layer_layout)


def init_params(cfg: ModelConfig, seed: int) -> Dict[object, torch.Tensor]:
    """fp32 flat buffers {layer index | 'embed' | 'head'} with the product's init."""
    p = {i: init_flat(layer_layout(cfg), "layer", i, cfg, seed) for i in range(cfg.n_layer)}
    p["embed"] = init_flat(embed_layout(cfg), "embed", 0, cfg, seed)
    p["head"] = init_flat(head_layout(cfg), "head", 0, cfg, seed)
    return p


def _gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _rope(t, S, theta=10000.0):
    """t: [n_seq, H, S, D]; rotate-half pairs (i, i+D/2), angle pos*theta^(-2i/D)."""
    D = t.shape[-1]
    half = D // 2
    inv = theta ** (-(2.0 * torch.arange(half, dtype=torch.float32)) / D)
    ang = torch.arange(S, dtype=torch.float32)[:, None] * inv[None, :]
    sn, cs = torch.sin(ang), torch.cos(ang)
    a, b = t[..., :half], t[..., half:]
    return torch.cat([a * cs - b * sn, a * sn + b * cs], -1)


def _attention(q, k, v, n_seq, S, H, D):
    s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    s = s.masked_fill(torch.ones(S, S, dtype=torch.bool).triu(1), float("-inf"))
    return (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(n_seq * S, H * D)


def _rmsnorm(x, w, eps=1e-5):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def _llama_block(cfg: ModelConfig, w, x, n_seq):
    S, H, D, f = cfg.seq_len, cfg.n_head, cfg.head_dim, cfg.ffn
    h = _rmsnorm(x, w["attn_norm"])
    q, k, v = (h @ w["qkv_w"].t()).view(n_seq, S, 3, H, D).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    q, k = _rope(q, S), _rope(k, S)
    x = x + _attention(q, k, v, n_seq, S, H, D) @ w["o_w"].t()
    gu = _rmsnorm(x, w["mlp_norm"]) @ w["gu_w"].t()
    return x + (F.silu(gu[:, :f]) * gu[:, f:]) @ w["down_w"].t()


def _block(cfg: ModelConfig, w, x, n_seq):
    if cfg.family == "llama":
        return _llama_block(cfg, w, x, n_seq)
    S, H, D, d = cfg.seq_len, cfg.n_head, cfg.head_dim, cfg.d_model
    h = F.layer_norm(x, (d,), w["ln1_w"], w["ln1_b"], 1e-5)
    qkv = h @ w["qkv_w"].t() + w["qkv_b"]
    q, k, v = qkv.view(n_seq, S, 3, H, D).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    s = (q @ k.transpose(-1, -2)) / math.sqrt(D)
    s = s.masked_fill(torch.ones(S, S, dtype=torch.bool).triu(1), float("-inf"))
    a = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(n_seq * S, d)
    x = x + a @ w["proj_w"].t() + w["proj_b"]
    h = F.layer_norm(x, (d,), w["ln2_w"], w["ln2_b"], 1e-5)
    g = _gelu(h @ w["fc1_w"].t() + w["fc1_b"])
    return x + g @ w["fc2_w"].t() + w["fc2_b"]


def loss_and_grads(cfg: ModelConfig, params: Dict[object, torch.Tensor], batch: torch.Tensor):
    """batch: [B, S+1] int tokens.  Returns (loss, {unit: fp32 grad flat})."""
    B = batch.shape[0]
    S = cfg.seq_len
    leaves = {k: v.detach().clone().requires_grad_() for k, v in params.items()}
    views = {k: (layer_layout(cfg) if isinstance(k, int) else
                 embed_layout(cfg) if k == "embed" else head_layout(cfg)).views(v)
             for k, v in leaves.items()}
    tok = batch[:, :S].reshape(-1).long()
    lab = batch[:, 1:].reshape(-1).long()
    e = views["embed"]
    x = e["wte"][tok]
    if "wpe" in e:
        x = x + e["wpe"][torch.arange(B * S) % S]
    for i in range(cfg.n_layer):
        x = _block(cfg, views[i], x, B)
    h = views["head"]
    if cfg.family == "llama":
        xf = _rmsnorm(x, h["norm_w"])
    else:
        xf = F.layer_norm(x, (cfg.d_model,), h["lnf_w"], h["lnf_b"], 1e-5)
    logits = xf @ h["head_w"].t()
    loss = F.cross_entropy(logits, lab, reduction="sum") / (B * S)
    loss.backward()
    return loss.item(), {k: v.grad for k, v in leaves.items()}


def adamw(params, grads, state, step, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, wd=0.1):
    """torch.optim.AdamW update rule, applied per flat buffer (in place)."""
    for k, p in params.items():
        g = grads[k]
        m, v = state.setdefault(k, (torch.zeros_like(p), torch.zeros_like(p)))
        p.mul_(1 - lr * wd)
        m.lerp_(g, 1 - beta1)
        v.mul_(beta2).addcmul_(g, g, value=1 - beta2)
        denom = (v.sqrt() / math.sqrt(1 - beta2 ** step)).add_(eps)
        p.addcdiv_(m, denom, value=-lr / (1 - beta1 ** step))


def train_steps(cfg: ModelConfig, batches, seed: int = 1234, **adam_kw):
    """Run len(batches) oracle steps; returns (losses, final params, last grads)."""
    params = init_params(cfg, seed)
    state: dict = {}
    losses = []
    grads = None
    for step, batch in enumerate(batches, start=1):
        loss, grads = loss_and_grads(cfg, params, batch)
        losses.append(loss)
        adamw(params, grads, state, step, **adam_kw)
    return losses, params, grads


def synthetic_batch(cfg: ModelConfig, global_batch: int, step: int, base_seed: int = 1234):
    from paper_2507_10392_b200.runtime.data import synthetic_batch as _sb
    return _sb(cfg.vocab, cfg.seq_len, global_batch, step, base_seed)
