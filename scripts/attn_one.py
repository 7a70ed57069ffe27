"""Run one attention fwd (tcgen05) + bwd at the GPT-2 small shape (for ncu)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
n, S, H, D = 8, 1024, 12, 64
qkv = torch.randn(n * S, 3 * H * D, device="cuda").bfloat16()
out = torch.empty(n * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n, H, S, device="cuda")
dout = torch.randn(n * S, H * D, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv); delta = torch.empty(n, H, S, device="cuda")
dq_acc = torch.empty(n * S, H * D, device="cuda")
for _ in range(2):
    K.attn_fwd(qkv, out, lse, n, S, H, D, 1 / math.sqrt(D))
    K.attn_bwd(qkv, out, dout, lse, dqkv, dq_acc, delta, n, S, H, D, 1 / math.sqrt(D))
torch.cuda.synchronize()
print("ok")
