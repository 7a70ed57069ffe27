"""TEST-ONLY torch-CPU twin of ``paper_2507_10392_b200.kernels``.

Same function names, argument meaning and in-place output contract as the
C-ABI kernels, computed in fp32 on CPU tensors.  It exists so the executor's
host logic (schedule walking, shard bookkeeping, routing, boundary transfers,
multi-rank collectives over gloo) can be exercised without a GPU.  The product
never imports this module (the product's kernels refuse CPU tensors).
"""

import math

import torch

EPI_BF16, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_GELU_BWD, EPI_F32, EPI_RESID, EPI_BIAS_GELU_NA = range(8)


def _gelu(x):
    return 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _gelu_grad(x):
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (x + k1 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * k0 * (1 + 3 * k1 * x * x)


def gemm(a, b, out, *, a_t=False, b_t=False, epilogue=EPI_BF16, bias=None, resid=None, aux=None,
         beta=0.0, M=None, N=None, K=None):
    A = a.float().t() if a_t else a.float()
    B = b.float() if b_t else b.float().t()
    acc = A @ B
    if epilogue == EPI_F32:
        out.copy_(acc + (beta * out if beta != 0.0 else 0.0))
        return out
    if epilogue in (EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_BIAS_GELU_NA):
        acc = acc + bias.float()
    if epilogue in (EPI_BIAS_RESID, EPI_RESID):
        acc = acc + resid.float()
    if epilogue == EPI_BIAS_GELU:
        aux.copy_(acc)
        acc = _gelu(aux.float())
    if epilogue == EPI_BIAS_GELU_NA:
        acc = _gelu(acc.bfloat16().float())
    if epilogue == EPI_GELU_BWD:
        acc = acc * _gelu_grad(aux.float())
    out.copy_(acc)
    return out


def layernorm_fwd(x, w, b, y, mean, rstd, eps=1e-5):
    xf = x.float()
    mu = xf.mean(-1)
    var = ((xf - mu[:, None]) ** 2).mean(-1)
    rs = torch.rsqrt(var + eps)
    y.copy_((xf - mu[:, None]) * rs[:, None] * w.float() + b.float())
    mean.copy_(mu)
    rstd.copy_(rs)


def layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=None, db_accum=None, db_out=None,
                  phase=0):
    xh = (x.float() - mean[:, None]) * rstd[:, None]
    if phase != 2:
        g = dy.float() * w.float()
        mg = g.mean(-1, keepdim=True)
        mgx = (g * xh).mean(-1, keepdim=True)
        out = rstd[:, None] * (g - mg - xh * mgx)
        if dx_accum is not None:
            out = out + dx_accum.float()
        dx.copy_(out)
    if phase == 1:
        return
    dw += (dy.float() * xh).sum(0)
    db += dy.float().sum(0)
    if db_accum is not None:
        db_accum += dx_accum.float().sum(0)
        db_out += dx.float().sum(0)


def embedding_fwd(tokens, wte, wpe, out, seq_len):
    pos = torch.arange(out.shape[0]) % seq_len
    x = wte.float()[tokens.long()]
    if wpe is not None:
        x = x + wpe.float()[pos]
    out.copy_(x)


def embedding_bwd(tokens, dout, dwte, dwpe, seq_len):
    pos = torch.arange(dout.shape[0]) % seq_len
    dwte.index_add_(0, tokens.long(), dout.float())
    if dwpe is not None:
        dwpe.index_add_(0, pos, dout.float())


def xent_fwd_bwd(logits, labels, loss_sum, dlogits, scale):
    lf = logits.float()
    lse = torch.logsumexp(lf, -1)
    lab = labels.long()
    ok = lab >= 0
    picked = lf.gather(1, lab.clamp(min=0)[:, None])[:, 0]
    loss_sum += ((lse - picked) * ok).sum()
    p = torch.softmax(lf, -1)
    p[torch.arange(p.shape[0]), lab.clamp(min=0)] -= 1.0
    dlogits.copy_(p * scale * ok[:, None])


def bias_grad(dy, db):
    db += dy.float().sum(0)


def _split(qkv, n_seq, S, H, D):
    q, k, v = qkv.float().view(n_seq, S, 3, H, D).unbind(2)
    return [t.transpose(1, 2) for t in (q, k, v)]


def attn_fwd(qkv, out, lse, n_seq, seq_len, n_head, head_dim, scale):
    q, k, v = _split(qkv, n_seq, seq_len, n_head, head_dim)
    s = (q @ k.transpose(-1, -2)) * scale
    mask = torch.ones(seq_len, seq_len, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse.copy_(torch.logsumexp(s, -1))
    o = torch.softmax(s, -1) @ v
    out.copy_(o.transpose(1, 2).reshape(n_seq * seq_len, n_head * head_dim))


def attn_bwd(qkv, out, dout, lse, dqkv, dq_accum, delta, n_seq, seq_len, n_head, head_dim, scale):
    qf = qkv.float().detach().requires_grad_()
    q, k, v = _split(qf, n_seq, seq_len, n_head, head_dim)
    s = (q @ k.transpose(-1, -2)) * scale
    mask = torch.ones(seq_len, seq_len, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    o = (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(n_seq * seq_len, n_head * head_dim)
    o.backward(dout.float())
    dqkv.copy_(qf.grad)


def adamw_shard(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, lr, beta1, beta2, eps,
                weight_decay, grad_scale, step):
    if isinstance(step, torch.Tensor):
        step = int(step.item())
    g = grad.float() * grad_scale
    if sumsq is not None:
        sumsq += (g * g).sum()
    master.mul_(1 - lr * weight_decay)
    exp_avg.lerp_(g, 1 - beta1)
    exp_avg_sq.mul_(beta2).addcmul_(g, g, value=1 - beta2)
    bc1 = 1 - beta1 ** step
    bc2 = 1 - beta2 ** step
    denom = (exp_avg_sq.sqrt() / math.sqrt(bc2)).add_(eps)
    master.addcdiv_(exp_avg, denom, value=-lr / bc1)
    param_bf16.copy_(master)


def embed_mark(tokens, rows, mark, step_dev):
    t = tokens.reshape(-1).long()
    t = t[(t >= 0) & (t < rows)]
    mark[t] = int(step_dev.reshape(-1)[0].item())


def embed_zero_rows(tokens, grad_table):
    t = tokens.reshape(-1).long()
    t = t[(t >= 0) & (t < grad_table.shape[0])]
    grad_table[t] = 0


def adamw_rows(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, mark, marked, lr, beta1,
               beta2, eps, weight_decay, grad_scale, step_dev):
    sel = (mark == int(step_dev.reshape(-1)[0].item())) == bool(marked)
    idx = sel.nonzero().reshape(-1)
    if idx.numel() == 0:
        return
    g = grad[idx] if marked else torch.zeros_like(master[idx])
    m_, a_, v_, p_ = master[idx], exp_avg[idx], exp_avg_sq[idx], param_bf16[idx]
    adamw_shard(m_, a_, v_, g, p_, sumsq if marked else None, lr, beta1, beta2, eps,
                weight_decay, grad_scale, step_dev)
    master[idx], exp_avg[idx], exp_avg_sq[idx], param_bf16[idx] = m_, a_, v_, p_


class GlooComm:
    """TEST-ONLY stand-in for runtime.comm.NcclComm over torch.distributed (gloo)."""

    def __init__(self, ranks, world_rank):
        import torch.distributed as dist

        self.dist = dist
        self.ranks = ranks
        self.rank = ranks.index(world_rank) if world_rank in ranks else -1
        self.pg = dist.new_group(ranks) if len(ranks) < dist.get_world_size() else None

    def allgather_v(self, buf, counts, displs):
        for r, (c, d) in enumerate(zip(counts, displs)):
            seg = buf[d:d + c]
            tmp = seg.float() if seg.dtype == torch.bfloat16 else seg
            self.dist.broadcast(tmp, src=self.ranks[r], group=self.pg)
            seg.copy_(tmp)

    def reduce_scatter_v(self, buf, counts, displs):
        for r, (c, d) in enumerate(zip(counts, displs)):
            seg = buf[d:d + c].clone()
            self.dist.reduce(seg, dst=self.ranks[r], group=self.pg)
            if r == self.rank:
                buf[d:d + c].copy_(seg)

    def p2p(self, ops):
        reqs = []
        tmps = []
        for peer, t, is_send in ops:
            if t.numel() == 0:
                continue
            f = t.float().contiguous()
            if is_send:
                reqs.append(self.dist.isend(f, peer))
            else:
                reqs.append(self.dist.irecv(f, peer))
                tmps.append((t, f))
        for r in reqs:
            r.wait()
        for t, f in tmps:
            t.copy_(f)

    def allreduce_sum(self, buf):
        self.dist.all_reduce(buf, group=self.pg)


class GlooGroupComm(GlooComm):
    """TEST-ONLY twin of runtime.comm.PeerGroup's interface over gloo: gather into a
    window slot, RS-v + AdamW on this rank's shard at the ReduceScatter event."""

    def gather(self, pu, dst, step_dev):
        dst[pu.lo:pu.hi].copy_(pu.shard)
        self.allgather_v(dst, pu.counts, pu.displs)

    def wait_consumed(self, pu, delta, step_dev):
        return None   # gloo collectives are synchronous

    def reduce_scatter_adamw(self, pu, adam, sumsq, step_dev, write_grad=False):
        self.reduce_scatter_v(pu.grad, pu.counts, pu.displs)
        adamw_shard(pu.master, pu.exp_avg, pu.exp_avg_sq, pu.grad[pu.lo:pu.hi], pu.shard,
                    sumsq, adam.lr, adam.beta1, adam.beta2, adam.eps, adam.weight_decay, 1.0,
                    step_dev)


def step_increment(step_dev):
    step_dev += 1


def rmsnorm_fwd(x, w, y, rstd, eps=1e-5):
    xf = x.float()
    rs = torch.rsqrt((xf * xf).mean(-1) + eps)
    y.copy_(xf * rs[:, None] * w.float())
    rstd.copy_(rs)


def rmsnorm_bwd(dy, x, w, rstd, dx, dw, dx_accum=None):
    xh = x.float() * rstd[:, None]
    g = dy.float() * w.float()
    out = rstd[:, None] * (g - xh * (g * xh).mean(-1, keepdim=True))
    if dx_accum is not None:
        out = out + dx_accum.float()
    dw += (dy.float() * xh).sum(0)
    dx.copy_(out)


def rope(qkv, seq_len, n_head, head_dim, theta=10000.0, inverse=False):
    rows = qkv.shape[0]
    half = head_dim // 2
    pos = (torch.arange(rows) % seq_len).float()
    inv = theta ** (-(2.0 * torch.arange(half).float()) / head_dim)
    ang = pos[:, None] * inv[None, :]
    sn, cs = torch.sin(ang), torch.cos(ang)
    if inverse:
        sn = -sn
    x = qkv[:, :2 * n_head * head_dim].float().view(rows, 2 * n_head, head_dim)
    a, b = x[..., :half], x[..., half:]
    na = a * cs[:, None, :] - b * sn[:, None, :]
    nb = a * sn[:, None, :] + b * cs[:, None, :]
    qkv[:, :2 * n_head * head_dim].copy_(torch.cat([na, nb], -1).view(rows, -1))


def swiglu_fwd(gu, out):
    f = out.shape[1]
    g, u = gu[:, :f].float(), gu[:, f:].float()
    out.copy_(torch.nn.functional.silu(g) * u)


def swiglu_bwd(gu, dout, dgu):
    f = dout.shape[1]
    g, u, d = gu[:, :f].float(), gu[:, f:].float(), dout.float()
    sg = torch.sigmoid(g)
    dg = d * u * sg * (1 + g * (1 - sg))
    du = d * g * sg
    dgu[:, :f].copy_(dg)
    dgu[:, f:].copy_(du)


def fill_f32(t, value):
    t.fill_(value)


def cast_f32_bf16(src, dst):
    dst.copy_(src)
