"""LayerNorm fwd / bwd at the GPT-2-small step shape, L2-warm (input just written,
as in the step) and L2-cold (a 256 MB buffer written between calls).
    python scripts/ln_warm_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K

T, d = 8192, 768
x = torch.randn(T, d, device="cuda").bfloat16()
w = torch.ones(d, device="cuda").bfloat16()
b = torch.zeros(d, device="cuda").bfloat16()
y = torch.empty_like(x)
mean = torch.empty(T, device="cuda")
rstd = torch.empty(T, device="cuda")
dy = torch.randn(T, d, device="cuda").bfloat16()
dx = torch.empty_like(x)
dw = torch.zeros(d, device="cuda")
db = torch.zeros(d, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, cold, iters=20):
    ts = []
    for i in range(iters + 3):
        if cold:
            flush.zero_()
        else:
            x.add_(0)  # rewrite the input: L2-resident like a producer's output
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


out = {}
for cold in (False, True):
    tag = "cold" if cold else "warm"
    us = timed(lambda: K.layernorm_fwd(x, w, b, y, mean, rstd), cold)
    out[f"ln_fwd_{tag}_us"] = round(us, 2)
    out[f"ln_fwd_{tag}_gbs"] = round(2 * T * d * 2 / us / 1e3)
    us = timed(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dy), cold)
    out[f"ln_bwd_{tag}_us"] = round(us, 2)
print(json.dumps(out))
