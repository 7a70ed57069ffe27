"""Time the step's GEMM shapes through one library build (A/B of kernel changes):
  python scripts/gemm_ab.py [path/to/libzorse_b200*.so]   -> one JSON line per shape"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_10392_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

from paper_2507_10392_b200 import kernels as K  # noqa: E402

T = 8192
SHAPES = [  # (name, M, N, K, kwargs builder)
    ("qkv fwd bias", T, 2304, 768, "bias"), ("proj fwd bias+resid", T, 768, 768, "bias_resid"),
    ("fc1 fwd bias+gelu(no aux)", T, 3072, 768, "gelu_na"), ("fc1 rc bias+gelu", T, 3072, 768, "gelu"),
    ("fc2 fwd bias+resid", T, 768, 3072, "bias_resid"), ("fc2 dgrad gelu'", T, 3072, 768, "gelu_bwd"),
    ("fc1 dgrad", T, 768, 3072, "dgrad"), ("qkv dgrad", T, 768, 2304, "dgrad"),
    ("fc1 wgrad", 3072, 768, T, "wgrad"), ("lm head", T, 50304, 768, "plain"),
    ("lm dgrad bf16", T, 768, 50304, "dgrad"), ("lm dgrad f32 split-K", T, 768, 50304, "dgrad_f32"),
]


def main():
    torch.manual_seed(0)
    out = []
    for name, M, N, Kd, kind in SHAPES:
        r = lambda *s: (torch.randn(*s, device="cuda") * 0.05).bfloat16()  # noqa: E731
        kw = {}
        if kind in ("dgrad", "dgrad_f32"):
            a, b = r(M, Kd), r(Kd, N)
            kw["b_t"] = True
            if kind == "dgrad_f32":
                kw.update(epilogue=K.EPI_F32, beta=1.0)
        elif kind == "wgrad":
            a, b = r(Kd, M), r(Kd, N)
            kw.update(a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0)
        else:
            a, b = r(M, Kd), r(N, Kd)
        o = torch.empty(M, N, device="cuda",
                        dtype=torch.float32 if kind in ("wgrad", "dgrad_f32") else torch.bfloat16)
        if kind in ("bias", "bias_resid", "gelu", "gelu_na"):
            kw["bias"] = r(N)
        if kind == "bias":
            kw["epilogue"] = K.EPI_BIAS
        if kind == "bias_resid":
            kw.update(epilogue=K.EPI_BIAS_RESID, resid=r(M, N))
        if kind == "gelu":
            kw.update(epilogue=K.EPI_BIAS_GELU, aux=torch.empty_like(o))
        if kind == "gelu_na":
            kw["epilogue"] = K.EPI_BIAS_GELU_NA
        if kind == "gelu_bwd":
            kw.update(epilogue=K.EPI_GELU_BWD, aux=r(M, N))
        fn = lambda: K.gemm(a, b, o, **kw)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                fn()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / 20)
        out.append({"gemm": name, "M": M, "N": N, "K": Kd, "us": best * 1e3,
                    "tile": K.gemm_choice(M, N, Kd, a_t=kw.get("a_t", False), b_t=kw.get("b_t", False),
                                          epilogue=kw.get("epilogue", 0), beta=kw.get("beta", 0.0)),
                    "tflops": 2 * M * N * Kd / (best * 1e-3) / 1e12})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
