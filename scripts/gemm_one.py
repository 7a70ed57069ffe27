import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
M = N = Kd = 8192
a = torch.randn(M, Kd, device="cuda").bfloat16(); b = torch.randn(N, Kd, device="cuda").bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3): K.gemm(a, b, out)
torch.cuda.synchronize(); print("ok")
