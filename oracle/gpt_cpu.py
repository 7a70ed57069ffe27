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
from dataclasses import dataclass
from typing import Dict, List, Tuple

import torch
import torch.nn.functional as F

# This module is self-contained: it imports nothing from the product package (so
# the CPU baseline / reference arm never loads the product's CUDA library).  The
# flat parameter layouts and the init rule below are the executor's documented
# contract, restated here independently; tests/test_parity_units.py
# pins the product's initial parameters bit-exactly against init_params().


@dataclass(frozen=True)
class OracleConfig:
    """Transformer shape (field meaning as the product's ModelConfig; any object
    with these attributes is accepted by the functions below)."""

    name: str
    family: str
    n_layer: int
    d_model: int
    n_head: int
    vocab: int
    seq_len: int
    d_ff: int = 0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head

    @property
    def ffn(self) -> int:
        return self.d_ff or 4 * self.d_model


GPT2_SMALL = OracleConfig("gpt2-small-124m", "gpt", 12, 768, 12, 50304, 1024)


def _ffn(cfg) -> int:
    return cfg.d_ff or 4 * cfg.d_model


def layer_entries(cfg) -> List[Tuple[str, Tuple[int, ...]]]:
    """Named tensors of one layer's flat buffer, in flat order."""
    d, f = cfg.d_model, _ffn(cfg)
    if cfg.family == "llama":
        return [("attn_norm", (d,)), ("qkv_w", (3 * d, d)), ("o_w", (d, d)),
                ("mlp_norm", (d,)), ("gu_w", (2 * f, d)), ("down_w", (d, f))]
    return [("ln1_w", (d,)), ("ln1_b", (d,)), ("qkv_w", (3 * d, d)), ("qkv_b", (3 * d,)),
            ("proj_w", (d, d)), ("proj_b", (d,)), ("ln2_w", (d,)), ("ln2_b", (d,)),
            ("fc1_w", (f, d)), ("fc1_b", (f,)), ("fc2_w", (d, f)), ("fc2_b", (d,))]


def embed_entries(cfg):
    if cfg.family == "llama":
        return [("wte", (cfg.vocab, cfg.d_model))]
    return [("wte", (cfg.vocab, cfg.d_model)), ("wpe", (cfg.seq_len, cfg.d_model))]


def head_entries(cfg):
    d = cfg.d_model
    if cfg.family == "llama":
        return [("norm_w", (d,)), ("head_w", (cfg.vocab, d))]
    return [("lnf_w", (d,)), ("lnf_b", (d,)), ("head_w", (cfg.vocab, d))]


def unit_entries(cfg, unit):
    """Entries of a unit: a layer index, "embed" or "head"."""
    if isinstance(unit, int):
        return layer_entries(cfg)
    return embed_entries(cfg) if unit == "embed" else head_entries(cfg)


def spans(entries):
    """[(name, lo, hi, shape)] flat element ranges."""
    out, off = [], 0
    for name, shape in entries:
        n = math.prod(shape)
        out.append((name, off, off + n, shape))
        off += n
    return out


def views(entries, flat: torch.Tensor) -> Dict[str, torch.Tensor]:
    return {name: flat[lo:hi].view(*shape) for name, lo, hi, shape in spans(entries)}


def _init_unit(cfg, entries, kind: str, index: int, seed: int) -> torch.Tensor:
    """GPT-2 init: N(0, 0.02) weights, residual projections (proj_w, fc2_w) N(0,
    0.02/sqrt(2L)), norm weights 1, biases 0; tensor t of a unit draws from its own
    CPU generator seeded seed*1000003 + kind*100003 + index*101 + t (kind: layer 0,
    embed 1, head 2)."""
    n = sum(math.prod(s) for _, s in entries)
    flat = torch.empty(n, dtype=torch.float32)
    resid_std = 0.02 / math.sqrt(2 * cfg.n_layer)
    kcode = {"layer": 0, "embed": 1, "head": 2}[kind]
    for t, (name, lo, hi, shape) in enumerate(spans(entries)):
        v = flat[lo:hi]
        if name.endswith("_b"):
            v.zero_()
        elif name.startswith("ln") or name.endswith("norm") or name == "norm_w":
            v.fill_(1.0)
        else:
            g = torch.Generator()
            g.manual_seed(seed * 1_000_003 + kcode * 100_003 + index * 101 + t)
            v.normal_(0.0, resid_std if name in ("proj_w", "fc2_w") else 0.02, generator=g)
    return flat


def init_params(cfg, seed: int) -> Dict[object, torch.Tensor]:
    """fp32 flat buffers {layer index | 'embed' | 'head'}."""
    p = {i: _init_unit(cfg, layer_entries(cfg), "layer", i, seed) for i in range(cfg.n_layer)}
    p["embed"] = _init_unit(cfg, embed_entries(cfg), "embed", 0, seed)
    p["head"] = _init_unit(cfg, head_entries(cfg), "head", 0, seed)
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
    S, H, D, f = cfg.seq_len, cfg.n_head, cfg.d_model // cfg.n_head, _ffn(cfg)
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
    S, H, D, d = cfg.seq_len, cfg.n_head, cfg.d_model // cfg.n_head, cfg.d_model
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
    vw = {k: views(unit_entries(cfg, k), v) for k, v in leaves.items()}
    tok = batch[:, :S].reshape(-1).long()
    lab = batch[:, 1:].reshape(-1).long()
    e = vw["embed"]
    x = e["wte"][tok]
    if "wpe" in e:
        x = x + e["wpe"][torch.arange(B * S) % S]
    for i in range(cfg.n_layer):
        x = _block(cfg, vw[i], x, B)
    h = vw["head"]
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


def synthetic_batch(cfg, global_batch: int, step: int, base_seed: int = 1234):
    """[global_batch, seq_len+1] int32 tokens ~ Uniform[0, vocab) from a CPU generator
    seeded base_seed + step (the executor's data contract)."""
    g = torch.Generator().manual_seed(base_seed + step)
    return torch.randint(0, cfg.vocab, (global_batch, cfg.seq_len + 1), generator=g,
                         dtype=torch.int32)
