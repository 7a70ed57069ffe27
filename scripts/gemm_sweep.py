"""Sweep tile configurations (1/2-CTA, BN, K-splits) over the step's GEMM shapes
(the library reads ZB_GEMM_CTAS / ZB_GEMM_BN / ZB_GEMM_SPLITS on every call)."""
import itertools, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_10392_b200 import kernels as K
from gemm_shapes import t_ms
SHAPES = [  # (name, M, N, K, layout, epilogue)
    ("fwd_qkv", 8192, 2304, 768, "tn", 1), ("fwd_proj", 8192, 768, 768, "tn", 3),
    ("fwd_fc1", 8192, 3072, 768, "tn", 2), ("fwd_fc2", 8192, 768, 3072, "tn", 3),
    ("dgrad_fc2", 8192, 3072, 768, "dgrad", 4), ("dgrad_fc1", 8192, 768, 3072, "dgrad", 0),
    ("dgrad_qkv", 8192, 768, 2304, "dgrad", 0), ("dgrad_proj", 8192, 768, 768, "dgrad", 0),
    ("wgrad_fc2", 768, 3072, 8192, "wgrad", 5), ("wgrad_fc1", 3072, 768, 8192, "wgrad", 5),
    ("wgrad_qkv", 2304, 768, 8192, "wgrad", 5), ("wgrad_proj", 768, 768, 8192, "wgrad", 5),
    ("head_fwd", 8192, 50304, 768, "tn", 0), ("head_dgrad", 8192, 768, 50304, "dgrad", 0),
    ("head_wgrad", 50304, 768, 8192, "wgrad", 5),
]
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
KEYS = ("ZB_GEMM_CTAS", "ZB_GEMM_BN", "ZB_GEMM_SPLITS")
for name, M, N, Kd, lay, epi in SHAPES:
    bias, aux = r(N), r(M, N)
    if lay == "tn":
        a, b, kw = r(M, Kd), r(N, Kd), {}
    elif lay == "dgrad":
        a, b, kw = r(M, Kd), r(Kd, N), {"b_t": True}
    else:
        a, b, kw = r(Kd, M), r(Kd, N), {"a_t": True, "b_t": True}
    if epi == 5:
        c = torch.zeros(M, N, device="cuda")
        kw.update(epilogue=5, beta=1.0)
    else:
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        kw.update(epilogue=epi)
        if epi in (1, 2, 3):
            kw["bias"] = bias
        if epi in (2, 4):
            kw["aux"] = aux
        if epi == 3:
            kw["resid"] = aux
    cfgs = [("auto", {})]
    for ctas, bn in itertools.product((1, 2), (128, 192, 256)):
        cfgs.append((f"{ctas}c_bn{bn}", {"ZB_GEMM_CTAS": str(ctas), "ZB_GEMM_BN": str(bn)}))
    if epi == 5:
        for ctas, bn, sp in itertools.product((1, 2), (128, 256), (1, 2, 3, 4, 6, 8)):
            cfgs.append((f"{ctas}c_bn{bn}_s{sp}", {"ZB_GEMM_CTAS": str(ctas), "ZB_GEMM_BN": str(bn),
                                                   "ZB_GEMM_SPLITS": str(sp)}))
    res = {"shape": name, "MNK": [M, N, Kd]}
    for cname, env in cfgs:
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        try:
            ms = t_ms(lambda: K.gemm(a, b, c, **kw), iters=20)
            res[cname] = round(2 * M * N * Kd / ms / 1e9)
        except Exception as exc:
            res[cname] = str(exc)[:60]
    for k in KEYS:
        os.environ.pop(k, None)
    print(json.dumps(res), flush=True)
