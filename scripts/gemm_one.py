"""One GEMM launch at a given shape / config, for ncu.
    python scripts/gemm_one.py M N K [tn|dgrad|wgrad] [epi]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
M, N, Kd = (int(x) for x in sys.argv[1:4])
lay = sys.argv[4] if len(sys.argv) > 4 else "tn"
epi = int(sys.argv[5]) if len(sys.argv) > 5 else 0
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
if lay == "tn":
    a, b, kw = r(M, Kd), r(N, Kd), {}
elif lay == "dgrad":
    a, b, kw = r(M, Kd), r(Kd, N), {"b_t": True}
else:
    a, b, kw = r(Kd, M), r(Kd, N), {"a_t": True, "b_t": True}
if epi == 5:
    c = torch.zeros(M, N, device="cuda"); kw.update(epilogue=5, beta=1.0)
else:
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); kw.update(epilogue=epi)
    if epi in (1, 2, 3, 7): kw["bias"] = r(N)
    if epi in (2, 4): kw["aux"] = r(M, N)
    if epi == 3: kw["resid"] = r(M, N)
for _ in range(3):
    K.gemm(a, b, c, **kw)
torch.cuda.synchronize()
print("ok")
