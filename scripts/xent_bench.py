"""Time the fused cross-entropy (loss + dlogits in place) at the LM-head shape.
  python scripts/xent_bench.py [LIB]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_10392_b200 import _lib
if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch
from paper_2507_10392_b200 import kernels as K

rows, V = 8192, 50304
logits = (3 * torch.randn(rows, V, device="cuda")).bfloat16()
labels = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
loss = torch.zeros(1, device="cuda")
work = logits.clone()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(12):
    work.copy_(logits)            # also flushes L2 (1.6 GB)
    torch.cuda.synchronize()
    s.record()
    K.xent_fwd_bwd(work, labels, loss, work, 1.0 / rows)
    e.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(s.elapsed_time(e))
us = sorted(ts)[len(ts) // 2] * 1e3
print(json.dumps({"xent_us": us, "tb_s": 2 * rows * V * 2 / us / 1e6, "lib": sys.argv[1] if len(sys.argv) > 1 else "new"}))
