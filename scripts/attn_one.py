"""One attention forward + backward at a given shape (for ncu captures).
  python scripts/attn_one.py [n_seq S H D]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2507_10392_b200 import kernels as K

n, S, H, D = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (8, 1024, 12, 64)))
T = n * S
torch.manual_seed(0)
qkv = torch.randn(T, 3 * H * D, device="cuda").bfloat16()
out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n, H, S, device="cuda")
dout = torch.randn(T, H * D, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
delta = torch.empty(n, H, S, device="cuda")
dq = torch.empty(T, H * D, device="cuda") if D == 64 else None
sc = 1 / math.sqrt(D)
for _ in range(3):
    K.attn_fwd(qkv, out, lse, n, S, H, D, sc)
    K.attn_bwd(qkv, out, dout, lse, dqkv, dq, delta, n, S, H, D, sc)
torch.cuda.synchronize()
print("attn_one ok")
