"""LM-head GEMMs (A = the [tokens, vocab] gradient, far larger than L2) under the
M-fastest and N-fastest tile rasters (ZB_GEMM_RASTER=0|1), vs cuBLAS.
    python scripts/gemm_raster_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K


def t_ms(fn, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


T, V, d = 8192, 50304, 768
dl = torch.randn(T, V, device="cuda").bfloat16()
w = torch.randn(V, d, device="cuda").bfloat16()
hf = torch.randn(T, d, device="cuda").bfloat16()
dx = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
dw = torch.zeros(V, d, device="cuda")
cases = {
    "dgrad 8192x768x50304": (lambda: K.gemm(dl, w, dx, b_t=True), lambda: torch.matmul(dl, w),
                             2.0 * T * d * V),
    "wgrad 50304x768x8192": (lambda: K.gemm(dl, hf, dw, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
                             lambda: torch.matmul(dl.t(), hf), 2.0 * T * d * V),
}
for name, (f, g, fl) in cases.items():
    row = {"gemm": name}
    for r in ("0", "1"):
        os.environ["ZB_GEMM_RASTER"] = r
        row[f"raster{r}_tflops"] = round(fl / t_ms(f) / 1e9)
    row["cublas_tflops"] = round(fl / t_ms(g) / 1e9)
    print(json.dumps(row), flush=True)
