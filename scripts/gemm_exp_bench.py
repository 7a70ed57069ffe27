"""1-CTA GEMM time at step shapes for the timing-experiment builds (ZB_GEMM_EXP:
1 = no output stores, 2 = no MMAs, 3 = no operand loads; pick the build with
ZB_LIB_PATH).  python scripts/gemm_exp_bench.py <label>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K


def t_us(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
os.environ["ZB_GEMM_CTAS"] = "1"
row = {"build": sys.argv[1] if len(sys.argv) > 1 else "product"}
for M, N, Kd, epi, bn in [(8192, 3072, 768, 1, 256), (8192, 3072, 768, 7, 256),
                          (8192, 2304, 768, 1, 256), (8192, 768, 3072, 3, 192),
                          (8192, 8192, 8192, 0, 256)]:
    os.environ["ZB_GEMM_BN"] = str(bn)
    a, b = r(M, Kd), r(N, Kd)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kw = {"epilogue": epi}
    if epi in (1, 3, 7):
        kw["bias"] = r(N)
    if epi == 3:
        kw["resid"] = r(M, N)
    row[f"{M}x{N}x{Kd}_e{epi}_us"] = round(t_us(lambda: K.gemm(a, b, c, **kw)), 1)
print(json.dumps(row), flush=True)
