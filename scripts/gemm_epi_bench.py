"""GEMM time per (tile config, epilogue) at the step's shapes, warm, back to back.
    python scripts/gemm_epi_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K


def t_ms(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
T = 8192
shapes = [(T, 3072, 768, "tn", [0, 1, 7, 2]), (T, 2304, 768, "tn", [0, 1]), (T, 768, 3072, "tn", [0, 3]),
          (T, 768, 768, "tn", [0, 3]), (T, 3072, 768, "dgrad", [0, 4]), (T, 768, 3072, "dgrad", [0]),
          (T, 768, 50304, "dgrad", [0])]
cfgs = [("1", "256"), ("1", "192"), ("1", "128"), ("2", "256"), ("2", "192"), ("4", "256"), ("4", "192")]
for M, N, Kd, lay, epis in shapes:
    if lay == "tn":
        a, b, kw0 = r(M, Kd), r(N, Kd), {}
    else:
        a, b, kw0 = r(M, Kd), r(Kd, N), {"b_t": True}
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    bias, aux, res = r(N), r(M, N), r(M, N)
    for epi in epis:
        kw = dict(kw0, epilogue=epi)
        if epi in (1, 2, 3, 7):
            kw["bias"] = bias
        if epi in (2, 4):
            kw["aux"] = aux
        if epi == 3:
            kw["resid"] = res
        row = {"shape": [M, N, Kd], "layout": lay, "epi": epi}
        for ctas, bn in cfgs:
            if ctas in ("2", "4") and bn == "192" and lay == "dgrad":
                continue
            os.environ["ZB_GEMM_CTAS"], os.environ["ZB_GEMM_BN"] = ctas, bn
            try:
                ms = t_ms(lambda: K.gemm(a, b, c, **kw))
                row[f"{ctas}cta_bn{bn}"] = round(2.0 * M * N * Kd / ms / 1e9)
            except Exception as ex:  # noqa: BLE001
                row[f"{ctas}cta_bn{bn}"] = str(ex)[:40]
        print(json.dumps(row), flush=True)
