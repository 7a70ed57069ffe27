"""One small call of every kernel family through the C ABI, for compute-sanitizer
(memcheck / synccheck / racecheck):

  compute-sanitizer --tool memcheck python scripts/sanitize_kernels.py

GEMM (every epilogue, 1-CTA / CTA-pair / multicast-pair tiles, K splits), attention
forward / backward (D 64 and 128, both forward kernels), LayerNorm / RMSNorm
forward+backward, RoPE, SwiGLU, embedding, cross-entropy, bias grad, AdamW, the
peer collectives on one device (G = 2 local arenas), and one training step of the
smoke model.  Exits 0 after printing "sanitize ok"."""
import ctypes
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2507_10392_b200 import kernels as K
from paper_2507_10392_b200._lib import call


def r(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).bfloat16()


def gemms():
    M, N, Kd = 512, 512, 256
    a, b, bias, res = r(M, Kd), r(N, Kd, scale=0.05), r(N), r(M, N)
    out, aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16), torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for pair in (0, 1, 2):
        for epi, kw in ((0, {}), (1, {"bias": bias}), (2, {"bias": bias, "aux": aux}),
                        (3, {"bias": bias, "resid": res}), (4, {"aux": aux}), (6, {"resid": res}),
                        (7, {"bias": bias})):
            K.gemm_tile(a, b, out, pair=pair, bn=256, epilogue=epi, **kw)
    c = torch.zeros(M, N, device="cuda")
    for splits in (1, 2):
        K.gemm_tile(r(Kd, M), r(Kd, N), c, a_t=True, b_t=True, epilogue=5, beta=1.0, splits=splits)
    K.gemm(a, r(Kd, N), out, b_t=True)
    K.gemm_tile(a, b, out, tma_epi=False, epilogue=1, bias=bias)


def attention():
    for n, S, H, D in ((1, 256, 2, 64), (1, 384, 2, 64), (1, 256, 2, 128), (1, 384, 1, 128)):
        T = n * S
        qkv = r(T, 3 * H * D)
        out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(n, H, S, device="cuda")
        K.attn_fwd(qkv, out, lse, n, S, H, D, 1 / math.sqrt(D))
        dqkv = torch.empty_like(qkv)
        delta = torch.empty(n, H, S, device="cuda")
        dq = torch.empty(T, H * D, device="cuda") if D == 64 else None
        K.attn_bwd(qkv, out, r(T, H * D), lse, dqkv, dq, delta, n, S, H, D, 1 / math.sqrt(D))


def elementwise():
    rows, d = 256, 768
    x, w, b = r(rows, d), r(d), r(d)
    y = torch.empty_like(x)
    mean, rstd = torch.empty(rows, device="cuda"), torch.empty(rows, device="cuda")
    K.layernorm_fwd(x, w, b, y, mean, rstd)
    dw, db = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
    dx = torch.empty_like(x)
    K.layernorm_bwd(r(rows, d), x, w, mean, rstd, dx, dw, db, dx_accum=r(rows, d))
    K.layernorm_bwd(r(rows, d), x, w, mean, rstd, dx, dw, db, dx_accum=r(rows, d),
                    db_accum=torch.zeros(d, device="cuda"), db_out=torch.zeros(d, device="cuda"))
    K.rmsnorm_fwd(x, w, y, rstd)
    K.rmsnorm_bwd(r(rows, d), x, w, rstd, dx, dw, dx_accum=r(rows, d))
    qkv = r(256, 3 * 256)
    K.rope(qkv, 128, 2, 128)
    K.rope(qkv, 128, 2, 128, inverse=True)
    gu = r(rows, 2 * 512)
    m = torch.empty(rows, 512, device="cuda", dtype=torch.bfloat16)
    K.swiglu_fwd(gu, m)
    K.swiglu_bwd(gu, m, gu)
    tok = torch.randint(0, 1000, (rows,), device="cuda", dtype=torch.int32)
    wte, wpe = r(1000, d), r(128, d)
    K.embedding_fwd(tok, wte, wpe, y, 128)
    K.embedding_bwd(tok, r(rows, d), torch.zeros(1000, d, device="cuda"),
                    torch.zeros(128, d, device="cuda"), 128)
    logits = r(rows, 1024)
    K.xent_fwd_bwd(logits, torch.randint(0, 1024, (rows,), device="cuda", dtype=torch.int32),
                   torch.zeros(1, device="cuda"), logits, 1.0 / rows)
    K.bias_grad(r(rows, 2304), torch.zeros(2304, device="cuda"))
    n = 100_003
    p = torch.randn(n, device="cuda")
    K.adamw_shard(p, torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda"),
                  torch.randn(n, device="cuda"), torch.empty(n, device="cuda", dtype=torch.bfloat16),
                  torch.zeros(1, device="cuda"), 1e-3, 0.9, 0.95, 1e-8, 0.1, 1.0, 1)


def peers():
    g, P = 2, 1 << 16
    counts, displs = [P // 2, P // 2], [0, P // 2]
    grad_off, shard_off = 256, 256 + 4 * P
    bufs = [torch.zeros(shard_off + P, dtype=torch.uint8, device="cuda") for _ in range(g)]
    bases = (ctypes.c_void_p * g)(*[x.data_ptr() for x in bufs])
    for x in bufs:
        x[:16].view(torch.int32)[:2] = 1
    ep = torch.tensor([1], dtype=torch.int32, device="cuda")
    st = torch.tensor([1], dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for me in range(g):
        dst = torch.empty(P, device="cuda", dtype=torch.bfloat16)
        for mode in (0, 1):
            call("zb_peer_allgather_v", bases, g, me, (ctypes.c_uint64 * g)(shard_off, shard_off),
                 dst.data_ptr(), 2, (ctypes.c_int64 * g)(*counts), (ctypes.c_int64 * g)(*displs),
                 0, ep.data_ptr(), -1, mode, s)
        n = counts[me]
        mstr, mm, vv = (torch.zeros(n, device="cuda") for _ in range(3))
        call("zb_peer_rs_adamw", bases, g, me, grad_off, displs[me], n, 0, ep.data_ptr(),
             mstr.data_ptr(), mm.data_ptr(), vv.data_ptr(),
             bufs[me][shard_off:shard_off + 2 * n].data_ptr(), None, None, 1e-3, 0.9, 0.95, 1e-8,
             0.1, 1.0, st.data_ptr(), s)
        call("zb_peer_wait", bases, g, me, 0, ep.data_ptr(), 0, s)


def main():
    torch.manual_seed(0)
    gemms()
    attention()
    elementwise()
    peers()
    torch.cuda.synchronize()
    import __graft_entry__
    __graft_entry__.smoke()
    torch.cuda.synchronize()
    print("sanitize ok", flush=True)


if __name__ == "__main__":
    main()
