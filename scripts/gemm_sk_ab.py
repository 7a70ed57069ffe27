"""Stream-K vs data-parallel 1-CTA tiles on the step's N = 768 GEMM shapes (TF/s).  The stream-K
kernel path was removed after this measurement; splits=-1 now keeps the default.
  python scripts/gemm_sk_ab.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_10392_b200 import kernels as K


def t_us(fn, iters=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


T = 8192
cases = [("proj fwd bias+resid", 768, 768, False, K.EPI_BIAS_RESID),
         ("fc2 fwd bias+resid", 768, 3072, False, K.EPI_BIAS_RESID),
         ("proj dgrad", 768, 768, True, K.EPI_BF16),
         ("qkv dgrad", 768, 2304, True, K.EPI_BF16),
         ("fc1 dgrad", 768, 3072, True, K.EPI_BF16)]
for name, N, Kd, b_t, epi in cases:
    a = torch.randn(T, Kd, device="cuda").bfloat16()
    b = (torch.randn(Kd, N, device="cuda") if b_t else torch.randn(N, Kd, device="cuda")).bfloat16()
    out = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    bias = torch.randn(N, device="cuda").bfloat16()
    r = torch.randn(T, N, device="cuda").bfloat16()
    kw = dict(b_t=b_t, epilogue=epi)
    if epi == K.EPI_BIAS_RESID:
        kw.update(bias=bias, resid=r)
    fl = 2.0 * T * N * Kd
    res = {"gemm": name}
    res["default_us"] = t_us(lambda: K.gemm(a, b, out, **kw))
    for bn in (192, 128, 256):
        res[f"dp{bn}_us"] = t_us(lambda: K.gemm_tile(a, b, out, pair=0, bn=bn, splits=0, **kw))
        res[f"sk{bn}_us"] = t_us(lambda: K.gemm_tile(a, b, out, pair=0, bn=bn, splits=-1, **kw))
    res = {k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}
    best = min((v, k) for k, v in res.items() if k.endswith("_us"))
    res["best"] = best[1]
    res["best_tflops"] = round(fl / best[0] / 1e6, 1)
    print(json.dumps(res), flush=True)
