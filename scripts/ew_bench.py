"""HBM-bound kernels of the step at GPT-2-small shapes: bias grad, LayerNorm, AdamW."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
from gemm_shapes import t_ms
T = 8192
out = {}
for n in (768, 2304, 3072):
    dy = torch.randn(T, n, device="cuda").bfloat16()
    db = torch.zeros(n, device="cuda")
    ms = t_ms(lambda: K.bias_grad(dy, db))
    out[f"bias_grad_{n}"] = {"us": round(ms * 1e3, 1), "gbs": round(T * n * 2 / ms / 1e6)}
n = 7087872
m, v, g, p = [torch.randn(n, device="cuda") for _ in range(4)]
pb = torch.empty(n, device="cuda", dtype=torch.bfloat16)
step = torch.ones(1, device="cuda", dtype=torch.int32)
ss = torch.zeros(1, device="cuda")
ms = t_ms(lambda: K.adamw_shard(p, m, v, g, pb, ss, 1e-3, 0.9, 0.95, 1e-8, 0.1, 1.0, step))
out["adamw_7.1M"] = {"us": round(ms * 1e3, 1), "gbs": round(n * 30 / ms / 1e6)}
print(json.dumps(out))
