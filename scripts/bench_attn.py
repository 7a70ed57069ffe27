"""Time the tcgen05 attention kernels at GPT-2 / Llama shapes (TF/s, causal FLOPs)."""
import sys, os, json, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_10392_b200 import _lib
if len(sys.argv) > 1:   # A/B: another library build
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
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

for (n, S, H, D) in [(8, 1024, 12, 64), (11, 1024, 12, 64), (2, 2048, 32, 128), (8, 1024, 25, 64)]:
    T = n * S
    qkv = torch.randn(T, 3 * H * D, device="cuda").bfloat16()
    out = torch.empty(T, H * D, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(n, H, S, device="cuda")
    dout = torch.randn(T, H * D, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv); delta = torch.empty(n, H, S, device="cuda")
    dq_acc = torch.empty(T, H * D, device="cuda")
    sc = 1 / math.sqrt(D)
    fl = 4.0 * n * H * S * S * D / 2
    r = {"shape": [n, S, H, D]}
    ms = t_ms(lambda: K.attn_fwd(qkv, out, lse, n, S, H, D, sc))
    r["fwd_ms"] = ms; r["fwd_tflops"] = fl / ms / 1e9
    ms = t_ms(lambda: K.attn_bwd(qkv, out, dout, lse, dqkv, dq_acc if D == 64 else None, delta, n, S, H, D, sc))
    r["bwd_ms"] = ms; r["bwd_tflops(2.5x fwd flops)"] = 2.5 * fl / ms / 1e9
    print(json.dumps(r), flush=True)
