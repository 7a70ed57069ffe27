"""Run the tcgen05 attention backward once at a small shape (hang/correctness probe)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
n, S, H, D = [int(x) for x in sys.argv[1:5]] if len(sys.argv) > 4 else (1, 128, 1, 64)
qkv = torch.randn(n * S, 3 * H * D, device="cuda").bfloat16()
out = torch.empty(n * S, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n, H, S, device="cuda")
dout = torch.randn(n * S, H * D, device="cuda").bfloat16()
dqkv = torch.zeros_like(qkv); delta = torch.empty(n, H, S, device="cuda")
K.attn_fwd(qkv, out, lse, n, S, H, D, 1 / math.sqrt(D))
torch.cuda.synchronize(); print("fwd ok", flush=True)
K.attn_bwd(qkv, out, dout, lse, dqkv, None, delta, n, S, H, D, 1 / math.sqrt(D))
torch.cuda.synchronize(); print("bwd ok", os.environ.get("ZB_ATTN_BWD_ONLY"), dqkv.float().abs().sum().item(), flush=True)
