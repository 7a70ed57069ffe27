"""Time the tcgen05 GEMM against torch.matmul (cuBLAS) at the training-step shapes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K

def t_ms(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

T = 8192
rows = []
for (M, N, Kd, lay) in [(T, 2304, 768, "tn"), (T, 768, 768, "tn"), (T, 3072, 768, "tn"), (T, 768, 3072, "tn"),
                        (T, 50304, 768, "tn"), (T, 768, 3072, "dgrad"), (T, 768, 50304, "dgrad"),
                        (3072, 768, T, "wgrad"), (50304, 768, T, "wgrad"), (8192, 8192, 8192, "tn")]:
    if lay == "tn":
        a = torch.randn(M, Kd, device="cuda").bfloat16(); b = torch.randn(N, Kd, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        f = lambda: K.gemm(a, b, out); g = lambda: torch.matmul(a, b.t())
    elif lay == "dgrad":
        a = torch.randn(M, Kd, device="cuda").bfloat16(); b = torch.randn(Kd, N, device="cuda").bfloat16()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        f = lambda: K.gemm(a, b, out, b_t=True); g = lambda: torch.matmul(a, b)
    else:
        a = torch.randn(Kd, M, device="cuda").bfloat16(); b = torch.randn(Kd, N, device="cuda").bfloat16()
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        f = lambda: K.gemm(a, b, out, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0); g = lambda: torch.matmul(a.t(), b)
    ms, ms_ref = t_ms(f), t_ms(g)
    fl = 2.0 * M * N * Kd
    rows.append(dict(shape=[M, N, Kd], layout=lay, ms=ms, tflops=fl / ms / 1e9, cublas_ms=ms_ref, cublas_tflops=fl / ms_ref / 1e9))
    print(json.dumps(rows[-1]), flush=True)
