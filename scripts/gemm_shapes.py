"""Per-shape timing of every GEMM of the GPT-2-small training step (8192 tokens),
with the epilogue the step uses, against torch.matmul (cuBLAS, plain bf16 out).

    python scripts/gemm_shapes.py            -> one JSON line per GEMM kind
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2507_10392_b200 import kernels as K


def t_ms(fn, iters=30, graph=True):
    """Device time per call: `iters` calls captured in one CUDA graph and replayed
    (no host launch gaps between short kernels), after eager warm-up."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if graph:
        g.replay()
    else:
        for _ in range(iters):
            fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    T, d, V = 8192, 768, 50304
    dev = "cuda"
    bf = dict(device=dev, dtype=torch.bfloat16)
    r = lambda *s: torch.randn(*s, device=dev).bfloat16()  # noqa: E731
    x, h4 = r(T, d), r(T, 4 * d)
    w_qkv, w_o, w_fc1, w_fc2, w_head = r(3 * d, d), r(d, d), r(4 * d, d), r(d, 4 * d), r(V, d)
    b3, b1, b4 = r(3 * d), r(d), r(4 * d)
    out3, out1, out4, aux4 = (torch.empty(T, 3 * d, **bf), torch.empty(T, d, **bf),
                              torch.empty(T, 4 * d, **bf), torch.empty(T, 4 * d, **bf))
    logits = torch.empty(T, V, **bf)
    dy1, dy3, dy4, dlog = r(T, d), r(T, 3 * d), r(T, 4 * d), r(T, V)
    g_qkv, g_o, g_fc1, g_fc2 = (torch.zeros(3 * d, d, device=dev), torch.zeros(d, d, device=dev),
                                torch.zeros(4 * d, d, device=dev), torch.zeros(d, 4 * d, device=dev))
    g_head = torch.zeros(V, d, device=dev)
    cases = [
        ("fwd qkv +bias", T, 3 * d, d, lambda: K.gemm(x, w_qkv, out3, epilogue=K.EPI_BIAS, bias=b3),
         lambda: torch.matmul(x, w_qkv.t())),
        ("fwd proj +bias+resid", T, d, d,
         lambda: K.gemm(x, w_o, out1, epilogue=K.EPI_BIAS_RESID, bias=b1, resid=x),
         lambda: torch.matmul(x, w_o.t())),
        ("fwd fc1 +bias+gelu", T, 4 * d, d,
         lambda: K.gemm(x, w_fc1, out4, epilogue=K.EPI_BIAS_GELU, bias=b4, aux=aux4),
         lambda: torch.matmul(x, w_fc1.t())),
        ("fwd fc2 +bias+resid", T, d, 4 * d,
         lambda: K.gemm(h4, w_fc2, out1, epilogue=K.EPI_BIAS_RESID, bias=b1, resid=x),
         lambda: torch.matmul(h4, w_fc2.t())),
        ("fwd head", T, V, d, lambda: K.gemm(x, w_head, logits), lambda: torch.matmul(x, w_head.t())),
        ("dgrad head", T, d, V, lambda: K.gemm(dlog, w_head, out1, b_t=True),
         lambda: torch.matmul(dlog, w_head)),
        ("dgrad fc2 +gelu'", T, 4 * d, d,
         lambda: K.gemm(dy1, w_fc2, out4, b_t=True, epilogue=K.EPI_GELU_BWD, aux=aux4),
         lambda: torch.matmul(dy1, w_fc2)),
        ("dgrad fc1", T, d, 4 * d, lambda: K.gemm(dy4, w_fc1, out1, b_t=True),
         lambda: torch.matmul(dy4, w_fc1)),
        ("dgrad qkv", T, d, 3 * d, lambda: K.gemm(dy3, w_qkv, out1, b_t=True),
         lambda: torch.matmul(dy3, w_qkv)),
        ("dgrad proj", T, d, d, lambda: K.gemm(dy1, w_o, out1, b_t=True),
         lambda: torch.matmul(dy1, w_o)),
        ("wgrad head", V, d, T,
         lambda: K.gemm(dlog, x, g_head, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
         lambda: torch.matmul(dlog.t(), x)),
        ("wgrad fc2", d, 4 * d, T,
         lambda: K.gemm(dy1, h4, g_fc2, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
         lambda: torch.matmul(dy1.t(), h4)),
        ("wgrad fc1", 4 * d, d, T,
         lambda: K.gemm(dy4, x, g_fc1, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
         lambda: torch.matmul(dy4.t(), x)),
        ("wgrad qkv", 3 * d, d, T,
         lambda: K.gemm(dy3, x, g_qkv, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
         lambda: torch.matmul(dy3.t(), x)),
        ("wgrad proj", d, d, T,
         lambda: K.gemm(dy1, x, g_o, a_t=True, b_t=True, epilogue=K.EPI_F32, beta=1.0),
         lambda: torch.matmul(dy1.t(), x)),
    ]
    tot_ours = tot_ref = 0.0
    for name, M, N, Kd, f, g in cases:
        ms, ms_ref = t_ms(f), t_ms(g)
        fl = 2.0 * M * N * Kd
        tot_ours += ms
        tot_ref += ms_ref
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": Kd, "us": round(ms * 1e3, 1),
                          "tflops": round(fl / ms / 1e9), "cublas_us": round(ms_ref * 1e3, 1),
                          "cublas_tflops": round(fl / ms_ref / 1e9)}), flush=True)
    print(json.dumps({"total_us_one_each": round(tot_ours * 1e3, 1),
                      "cublas_total_us": round(tot_ref * 1e3, 1)}))


if __name__ == "__main__":
    main()
