"""LayerNorm fwd / bwd-dx / full bwd timing at the step's shape (8192 x 768), warm
(L2-resident inputs, as in the step) and cold (a 256 MB buffer written between calls).
  python scripts/ln_bench.py [path/to/libzorse_b200*.so]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_10392_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

from paper_2507_10392_b200 import kernels as K  # noqa: E402

T, d = 8192, 768
x, dy, dres = [torch.randn(T, d, device="cuda").bfloat16() for _ in range(3)]
w, b = torch.randn(d, device="cuda").bfloat16(), torch.randn(d, device="cuda").bfloat16()
y, dx = torch.empty_like(x), torch.empty_like(x)
mean, rstd = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
dw, db = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t_us(fn, cold):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(20):
        if cold:
            flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        ev.append((s, e))
    torch.cuda.synchronize()
    return sorted(s.elapsed_time(e) for s, e in ev)[len(ev) // 2] * 1e3


out = {"lib": os.path.basename(_lib.LIB_PATH)}
for cold in (False, True):
    tag = "cold" if cold else "warm"
    f = t_us(lambda: K.layernorm_fwd(x, w, b, y, mean, rstd), cold)
    bx = t_us(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres, phase=1), cold)
    bw = t_us(lambda: K.layernorm_bwd(dy, x, w, mean, rstd, dx, dw, db, dx_accum=dres), cold)
    out.update({f"fwd_us_{tag}": round(f, 2), f"fwd_gbs_{tag}": round(T * d * 4 / f / 1e3),
                f"bwd_dx_us_{tag}": round(bx, 2), f"bwd_dx_gbs_{tag}": round(T * d * 8 / bx / 1e3),
                f"bwd_us_{tag}": round(bw, 2)})
print(json.dumps(out))
