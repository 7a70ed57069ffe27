"""Column reductions of the step (bias grads 8192x3072 / 8192x2304, LayerNorm backward
with the folded bias grads), cold: a 512 MB buffer is READ between calls (a write-flush
would leave L2 full of dirty lines whose write-back the timed kernel would pay for).
  python scripts/colred_bench.py [LIB]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_10392_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch
from paper_2507_10392_b200 import kernels as K
flush = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
sink = torch.zeros(1, device="cuda")
T, d = 8192, 768


def t_us(fn):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(15):
        torch.sum(flush, dim=0, keepdim=True, out=sink)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record()
        ev.append((s, e))
    torch.cuda.synchronize()
    return sorted(s.elapsed_time(e) for s, e in ev)[len(ev) // 2] * 1e3


out = {"lib": os.path.basename(_lib.LIB_PATH)}
for n in (3072, 2304):
    dy = torch.randn(T, n, device="cuda").bfloat16()
    db = torch.zeros(n, device="cuda")
    us = t_us(lambda: K.bias_grad(dy, db))
    out[f"bias_grad_{n}_us"] = round(us, 2)
    out[f"bias_grad_{n}_tbs"] = round(T * n * 2 / us / 1e6, 2)
x, dy, dres, dxo = [torch.randn(T, d, device="cuda").bfloat16() for _ in range(4)]
w = torch.randn(d, device="cuda").bfloat16()
mean, rstd = torch.zeros(T, device="cuda"), torch.ones(T, device="cuda")
dw, db, dbr, dbo = [torch.zeros(d, device="cuda") for _ in range(4)]
dx = torch.empty_like(x)
out["ln_bwd_ex_us"] = round(t_us(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres,
                                                        db_accum=dbr, db_out=dbo)), 2)
out["ln_bwd_us"] = round(t_us(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db)), 2)
print(json.dumps(out))
