"""Per-kernel numerics vs plain torch fp32 references of the same op (GPU only)."""

import math

import pytest
import torch

from paper_2507_10392_b200 import kernels as K

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / (b.norm() + 1e-12)).item()


@pytest.mark.parametrize("rows,d", [(256, 256), (1000, 768), (64, 1600), (33, 5120)])
def test_layernorm_fwd_bwd(cuda, rows, d):
    torch.manual_seed(0)
    x = torch.randn(rows, d, device="cuda").bfloat16()
    w = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    b = (0.1 * torch.randn(d, device="cuda")).bfloat16()
    y = torch.empty_like(x)
    mean = torch.empty(rows, device="cuda")
    rstd = torch.empty(rows, device="cuda")
    K.layernorm_fwd(x, w, b, y, mean, rstd)
    xf = x.float().requires_grad_()
    wf = w.float().requires_grad_()
    bf = b.float().requires_grad_()
    ref = torch.nn.functional.layer_norm(xf, (d,), wf, bf, 1e-5)
    assert rel(y, ref) < 1e-2
    dy = torch.randn(rows, d, device="cuda").bfloat16()
    dres = torch.randn(rows, d, device="cuda").bfloat16()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dw = torch.zeros(d, device="cuda")
    db = torch.zeros(d, device="cuda")
    K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres)
    torch.cuda.synchronize()
    assert rel(dx, xf.grad + dres.float()) < 1e-2
    assert rel(dw, wf.grad) < 1e-3
    assert rel(db, bf.grad) < 1e-3
    # folded bias gradients: column sums of the residual grad and of the output
    dw.zero_(); db.zero_()
    db_res = torch.full((d,), 0.5, device="cuda")
    db_out = torch.full((d,), -0.25, device="cuda")
    K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres, db_accum=db_res, db_out=db_out)
    torch.cuda.synchronize()
    assert rel(dw, wf.grad) < 1e-3 and rel(db, bf.grad) < 1e-3
    assert rel(db_res, 0.5 + dres.float().sum(0)) < 1e-3
    assert rel(db_out, -0.25 + dx.float().sum(0)) < 1e-3
    # the same split in its two launches (zb_layernorm_bwd_phase 1 then 2)
    dx2 = torch.empty_like(x)
    dw2, db2 = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
    db_res2, db_out2 = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
    for ph in (1, 2):
        K.layernorm_bwd(dy, x, w, mean, rstd, dx2, dw2, db2, dx_accum=dres, db_accum=db_res2,
                        db_out=db_out2, phase=ph)
    torch.cuda.synchronize()
    assert torch.equal(dx2, dx)
    assert rel(dw2, wf.grad) < 1e-3 and rel(db2, bf.grad) < 1e-3
    assert rel(db_res2, dres.float().sum(0)) < 1e-3
    assert rel(db_out2, dx.float().sum(0)) < 1e-3


def test_embedding(cuda):
    torch.manual_seed(1)
    V, d, S, n = 1000, 256, 128, 3
    wte = torch.randn(V, d, device="cuda").bfloat16()
    wpe = torch.randn(S, d, device="cuda").bfloat16()
    tok = torch.randint(0, V, (n * S,), device="cuda", dtype=torch.int32)
    out = torch.empty(n * S, d, device="cuda", dtype=torch.bfloat16)
    K.embedding_fwd(tok, wte, wpe, out, S)
    pos = torch.arange(n * S, device="cuda") % S
    ref = wte.float()[tok.long()] + wpe.float()[pos]
    assert rel(out, ref) < 1e-2
    g = torch.randn(n * S, d, device="cuda").bfloat16()
    dwte = torch.zeros(V, d, device="cuda")
    dwpe = torch.zeros(S, d, device="cuda")
    K.embedding_bwd(tok, g, dwte, dwpe, S)
    rte = torch.zeros(V, d, device="cuda").index_add_(0, tok.long(), g.float())
    rpe = torch.zeros(S, d, device="cuda").index_add_(0, pos, g.float())
    torch.cuda.synchronize()
    assert rel(dwte, rte) < 1e-5 and rel(dwpe, rpe) < 1e-5


@pytest.mark.parametrize("rows,V", [(64, 50304), (300, 32000), (7, 1024)])
def test_xent(cuda, rows, V):
    torch.manual_seed(2)
    logits = (3 * torch.randn(rows, V, device="cuda")).bfloat16()
    labels = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    labels[0] = -1  # ignored row
    loss = torch.zeros(1, device="cuda")
    scale = 1.0 / 777
    g = torch.empty_like(logits)
    K.xent_fwd_bwd(logits, labels, loss, g, scale)
    lf = logits.float().requires_grad_()
    ref = torch.nn.functional.cross_entropy(lf, labels.long(), ignore_index=-1, reduction="sum")
    (ref * scale).backward()
    torch.cuda.synchronize()
    assert abs(loss.item() - ref.item()) / abs(ref.item()) < 1e-4
    assert rel(g, lf.grad) < 1e-2
    assert g[0].float().abs().max().item() == 0.0


def test_bias_grad(cuda):
    torch.manual_seed(3)
    dy = torch.randn(5000, 2304, device="cuda").bfloat16()
    db = torch.ones(2304, device="cuda")
    K.bias_grad(dy, db)
    torch.cuda.synchronize()
    assert rel(db, 1 + dy.float().sum(0)) < 1e-5


def _attn_ref(qkv, n_seq, S, H, D):
    q, k, v = qkv.float().view(n_seq, S, 3, H, D).unbind(2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))  # [n, H, S, D]
    s = q @ k.transpose(-1, -2) / math.sqrt(D)
    mask = torch.ones(S, S, device=qkv.device, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(n_seq * S, H * D), lse


@pytest.mark.parametrize("bwd", ["two-pass", "fused-dq"])
@pytest.mark.parametrize("n_seq,S,H,D", [(2, 128, 4, 64), (1, 1024, 3, 64), (2, 256, 2, 128),
                                         (1, 2048, 2, 128), (3, 512, 12, 64), (1, 384, 2, 128),
                                         (2, 768, 3, 64), (1, 2048, 5, 64)])
def test_attention_fwd_bwd(cuda, n_seq, S, H, D, bwd):
    """tcgen05 attention vs torch fp32: forward kernels by S % 256 (query-tile pairs,
    else the 2-CTA/SM (D 64) or single-tile (D 128) kernel); backward fused (dQ
    reduce-added, D = 64) or two passes."""
    fused = bwd == "fused-dq"
    torch.manual_seed(4)
    T = n_seq * S
    qkv = torch.randn(T, 3 * H * D, device="cuda").bfloat16()
    out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(n_seq, H, S, device="cuda")
    scale = 1.0 / math.sqrt(D)
    K.attn_fwd(qkv, out, lse, n_seq, S, H, D, scale)
    qf = qkv.float().requires_grad_()
    ro, rlse = _attn_ref(qf, n_seq, S, H, D)
    torch.cuda.synchronize()
    assert rel(out, ro) < 1e-2
    assert (lse - rlse).abs().max().item() < 1e-2
    dout = torch.randn(T, H * D, device="cuda").bfloat16()
    ro.backward(dout.float())
    dqkv = torch.empty_like(qkv)
    delta = torch.empty(n_seq, H, S, device="cuda")
    dq_acc = torch.empty(T, H * D, device="cuda") if fused else None
    K.attn_bwd(qkv, out, dout, lse, dqkv, dq_acc, delta, n_seq, S, H, D, scale)
    torch.cuda.synchronize()
    g = qf.grad.view(T, 3, H * D)
    d = dqkv.view(T, 3, H * D)
    assert rel(d[:, 0], g[:, 0]) < 2e-2, "dQ"
    assert rel(d[:, 1], g[:, 1]) < 2e-2, "dK"
    assert rel(d[:, 2], g[:, 2]) < 2e-2, "dV"


def test_adamw_matches_torch(cuda):
    torch.manual_seed(5)
    n = 100_003
    p = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    ref = p.clone().requires_grad_()
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    pb = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    ss = torch.zeros(1, device="cuda")
    for step in (1, 2, 3):
        ref.grad = g * step
        opt.step()
        K.adamw_shard(p, m, v, g * step, pb, ss, 1e-3, 0.9, 0.95, 1e-8, 0.1, 1.0, step)
    torch.cuda.synchronize()
    assert (p - ref.detach()).abs().max().item() < 1e-6
    assert rel(pb, ref.detach()) < 1e-2
    assert abs(ss.item() - sum(((g * s) ** 2).sum().item() for s in (1, 2, 3))) / ss.item() < 1e-4


def test_row_split_embedding_adamw_bit_exact(cuda):
    """Row-split token-embedding update (executor.sparse_embed): unmarked rows with g = 0
    early, marked rows after the backward == the dense AdamW over a gradient that is zero
    outside the tokens' rows, bit for bit; the token rows of the gradient are cleared."""
    torch.manual_seed(9)
    V, d, n_tok = 5003, 768, 4096
    tok = torch.randint(0, V, (2, n_tok // 2), device="cuda", dtype=torch.int32)
    step = torch.tensor([3], device="cuda", dtype=torch.int32)
    mark = torch.zeros(V, device="cuda", dtype=torch.int32)
    mark[:7] = 2                                   # stale marks of an earlier step
    st = {k: torch.randn(V, d, device="cuda") for k in ("p", "m")}
    st["v"] = torch.rand(V, d, device="cuda")
    grad = torch.randn(V, d, device="cuda")        # stale slot contents
    dense = {k: t.clone() for k, t in st.items()}
    K.embed_mark(tok, V, mark, step)
    K.embed_zero_rows(tok, grad)
    rows = torch.unique(tok.long())
    assert torch.equal(mark == 3, torch.zeros(V, dtype=torch.bool, device="cuda").index_fill_(0, rows, True))
    assert grad[rows].abs().max().item() == 0.0
    upd = torch.randn(rows.numel(), d, device="cuda")
    grad[rows] += upd                              # the embedding backward's scatter-add
    gd = torch.zeros(V, d, device="cuda")
    gd[rows] = grad[rows]
    pb, pbd = torch.empty(V, d, device="cuda", dtype=torch.bfloat16), torch.empty(V, d, device="cuda", dtype=torch.bfloat16)
    ss, ssd = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    hp = (1e-3, 0.9, 0.95, 1e-8, 0.1, 1.0)
    K.adamw_rows(st["p"], st["m"], st["v"], None, pb, ss, mark, False, *hp, step)
    K.adamw_rows(st["p"], st["m"], st["v"], grad, pb, ss, mark, True, *hp, step)
    K.adamw_shard(dense["p"], dense["m"], dense["v"], gd, pbd, ssd, *hp, step)
    torch.cuda.synchronize()
    for k in st:
        assert torch.equal(st[k], dense[k]), k
    assert torch.equal(pb, pbd)
    assert abs(ss.item() - ssd.item()) <= 1e-5 * ssd.item()


@pytest.mark.parametrize("rows,d", [(300, 512), (64, 4096), (17, 5120)])
def test_rmsnorm(cuda, rows, d):
    torch.manual_seed(6)
    x = torch.randn(rows, d, device="cuda").bfloat16()
    w = (1 + 0.1 * torch.randn(d, device="cuda")).bfloat16()
    y = torch.empty_like(x)
    rstd = torch.empty(rows, device="cuda")
    K.rmsnorm_fwd(x, w, y, rstd)
    xf = x.float().requires_grad_()
    wf = w.float().requires_grad_()
    ref = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + 1e-5) * wf
    assert rel(y, ref) < 1e-2
    dy = torch.randn(rows, d, device="cuda").bfloat16()
    dres = torch.randn(rows, d, device="cuda").bfloat16()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dw = torch.zeros(d, device="cuda")
    K.rmsnorm_bwd(dy, x, w, rstd, dx, dw, dx_accum=dres)
    torch.cuda.synchronize()
    assert rel(dx, xf.grad + dres.float()) < 1e-2
    assert rel(dw, wf.grad) < 1e-3


@pytest.mark.parametrize("n,S,H,D", [(2, 128, 4, 128), (1, 2048, 2, 128), (2, 256, 3, 64)])
def test_rope_roundtrip_and_reference(cuda, n, S, H, D):
    torch.manual_seed(7)
    qkv = torch.randn(n * S, 3 * H * D, device="cuda").bfloat16()
    orig = qkv.clone()
    K.rope(qkv, S, H, D)
    half = D // 2
    inv = 10000.0 ** (-(2.0 * torch.arange(half, device="cuda").float()) / D)
    ang = (torch.arange(n * S, device="cuda") % S).float()[:, None] * inv[None]
    x = orig[:, :2 * H * D].float().view(n * S, 2 * H, D)
    a, b = x[..., :half], x[..., half:]
    sn, cs = torch.sin(ang)[:, None], torch.cos(ang)[:, None]
    ref = torch.cat([a * cs - b * sn, a * sn + b * cs], -1).view(n * S, -1)
    torch.cuda.synchronize()
    assert rel(qkv[:, :2 * H * D], ref) < 1e-2
    assert torch.equal(qkv[:, 2 * H * D:], orig[:, 2 * H * D:])  # v untouched
    K.rope(qkv, S, H, D, inverse=True)
    torch.cuda.synchronize()
    assert rel(qkv, orig) < 1e-2


def test_swiglu(cuda):
    torch.manual_seed(8)
    rows, f = 257, 1376
    gu = torch.randn(rows, 2 * f, device="cuda").bfloat16()
    out = torch.empty(rows, f, device="cuda", dtype=torch.bfloat16)
    K.swiglu_fwd(gu, out)
    g = gu.float().requires_grad_()
    ref = torch.nn.functional.silu(g[:, :f]) * g[:, f:]
    assert rel(out, ref) < 1e-2
    d = torch.randn(rows, f, device="cuda").bfloat16()
    ref.backward(d.float())
    dgu = gu.clone()
    K.swiglu_bwd(dgu, d, dgu)  # in place
    torch.cuda.synchronize()
    assert rel(dgu, g.grad) < 1e-2


def test_gemm_resid_epilogue(cuda):
    torch.manual_seed(9)
    a = torch.randn(384, 512, device="cuda").bfloat16()
    b = (0.05 * torch.randn(640, 512, device="cuda")).bfloat16()
    r = torch.randn(384, 640, device="cuda").bfloat16()
    out = torch.empty(384, 640, device="cuda", dtype=torch.bfloat16)
    K.gemm(a, b, out, epilogue=K.EPI_RESID, resid=r)
    torch.cuda.synchronize()
    assert rel(out, a.float() @ b.float().t() + r.float()) < 1e-2
