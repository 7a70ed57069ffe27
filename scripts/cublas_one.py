"""One cuBLAS (torch.matmul) launch at a GEMM shape, for ncu comparisons.
    python scripts/cublas_one.py M N K [tn|dgrad|wgrad]"""
import sys
import torch
M, N, Kd = (int(x) for x in sys.argv[1:4])
lay = sys.argv[4] if len(sys.argv) > 4 else "tn"
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
if lay == "tn":
    a, b = r(M, Kd), r(N, Kd).t()
elif lay == "dgrad":
    a, b = r(M, Kd), r(Kd, N)
else:
    a, b = r(Kd, M).t(), r(Kd, N)
for _ in range(3):
    c = torch.matmul(a, b)
torch.cuda.synchronize()
print("ok")
