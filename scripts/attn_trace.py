"""Attention forward phase trace (debug build with -DZB_EXP_TRACE): per-role cycle totals.
  python scripts/attn_trace.py LIB [n_seq S H D]"""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_10392_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch
from paper_2507_10392_b200 import kernels as K
n, S, H, D = (int(x) for x in (sys.argv[2:6] if len(sys.argv) >= 6 else (8, 1024, 12, 64)))
T = n * S
torch.manual_seed(0)
qkv = torch.randn(T, 3 * H * D, device="cuda").bfloat16()
out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n, H, S, device="cuda")
dout = torch.randn(T, H * D, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
delta = torch.empty(n, H, S, device="cuda")
dq = torch.empty(T, H * D, device="cuda") if D == 64 else None
bwd = os.environ.get("TRACE_BWD") == "1"
for i in range(2):
    print(f"=== launch {i}", flush=True)
    K.attn_fwd(qkv, out, lse, n, S, H, D, 1 / math.sqrt(D))
    torch.cuda.synchronize()
    if bwd:
        print(f"=== bwd launch {i}", flush=True)
        K.attn_bwd(qkv, out, dout, lse, dqkv, dq, delta, n, S, H, D, 1 / math.sqrt(D))
        torch.cuda.synchronize()
