"""Graph-timed sweep of explicit tiles for given step GEMM shapes (interleaved repeats,
median), to check / refresh gemm_tune_cache.txt entries.
  python scripts/gemm_tile_sweep.py"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2507_10392_b200 import kernels as K


def graph_us(fn, iters=20):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


T = 8192
shapes = [("dgrad fc1", T, 768, 3072, "dgrad", K.EPI_BF16), ("dgrad qkv", T, 768, 2304, "dgrad", K.EPI_BF16),
          ("fwd fc2 +bias+resid", T, 768, 3072, "tn", K.EPI_BIAS_RESID),
          ("dgrad proj", T, 768, 768, "dgrad", K.EPI_BF16), ("fwd proj +bias+resid", T, 768, 768, "tn", K.EPI_BIAS_RESID)]
cands = [(0, 192), (0, 256), (0, 128), (1, 256), (1, 192), (2, 256)]
for name, M, N, Kd, lay, epi in shapes:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    b = (torch.randn(Kd, N, device="cuda") if lay == "dgrad" else torch.randn(N, Kd, device="cuda")).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    kw = dict(b_t=lay == "dgrad", epilogue=epi)
    if epi == K.EPI_BIAS_RESID:
        kw.update(bias=torch.randn(N, device="cuda").bfloat16(), resid=torch.randn(M, N, device="cuda").bfloat16())
    res = {}
    for rep in range(3):
        for pair, bn in cands:
            try:
                t = graph_us(lambda: K.gemm_tile(a, b, out, pair=pair, bn=bn, splits=1, **kw))
            except Exception as ex:  # unsupported layout for this tile
                continue
            res.setdefault(f"p{pair}b{bn}", []).append(t)
        res.setdefault("default", []).append(graph_us(lambda: K.gemm(a, b, out, **kw)))
        cb = torch.randn(M, Kd, device="cuda").bfloat16()
        res.setdefault("cublas", []).append(graph_us(lambda: torch.matmul(a, b if lay == "dgrad" else b.t())))
    med = {k: round(sorted(v)[len(v) // 2], 2) for k, v in res.items()}
    print(json.dumps({"gemm": name, "choice": K.gemm_choice(M, N, Kd, b_t=lay == "dgrad", epilogue=epi), **med}), flush=True)
