"""Mainloop efficiency per operand layout (TN / dgrad / wgrad) at a few sizes."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
from gemm_shapes import t_ms
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
for (M, N, Kd) in [(8192, 8192, 8192), (4096, 4096, 8192), (3072, 768, 8192), (768, 3072, 8192), (2304, 768, 8192)]:
    out = {"M": M, "N": N, "K": Kd, "ctas": os.environ.get("ZB_GEMM_CTAS", "auto")}
    a, b = r(M, Kd), r(N, Kd)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    out["tn"] = round(2 * M * N * Kd / t_ms(lambda: K.gemm(a, b, c)) / 1e9)
    bt = r(Kd, N)
    out["dgrad"] = round(2 * M * N * Kd / t_ms(lambda: K.gemm(a, bt, c, b_t=True)) / 1e9)
    at = r(Kd, M)
    cf = torch.zeros(M, N, device="cuda")
    out["wgrad_b0"] = round(2 * M * N * Kd / t_ms(lambda: K.gemm(at, bt, cf, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=0.0)) / 1e9)
    out["wgrad_b1"] = round(2 * M * N * Kd / t_ms(lambda: K.gemm(at, bt, cf, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0)) / 1e9)
    out["cublas_tn"] = round(2 * M * N * Kd / t_ms(lambda: torch.matmul(a, b.t())) / 1e9)
    out["cublas_wgrad"] = round(2 * M * N * Kd / t_ms(lambda: torch.matmul(at.t(), bt)) / 1e9)
    print(json.dumps(out), flush=True)
