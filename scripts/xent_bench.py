"""Fused cross-entropy (loss + dlogits in place) at the GPT-2-small LM-head shape.
    python scripts/xent_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K

T, V = 8192, 50304
logits = torch.randn(T, V, device="cuda").bfloat16()
labels = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
loss = torch.zeros(1, device="cuda")
for _ in range(2):
    K.xent_fwd_bwd(logits, labels, loss, logits, 1.0 / T)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    K.xent_fwd_bwd(logits, labels, loss, logits, 1.0 / T)
e.record()
torch.cuda.synchronize()
us = s.elapsed_time(e) / 10 * 1e3
print(json.dumps({"xent_us": round(us, 1), "hbm_gbs_1r1w": round(2 * T * V * 2 / us / 1e3)}))
