"""Profile ingestion: measure one transformer layer's forward
and backward (gradient pass only — recompute is charged separately, as in the
reference's fixtures.py:37-41) on this B200 at per-device batches 1/2/4/8
sequences, and emit a cluster-profile JSON (docs/file_formats.md:7-36) whose
runtime_samples are MEASURED ("b200") plus an emulated half-speed kind
("b200h" = 2x).  Then plan_training runs on it.

  python scripts/profile_layers.py [model] [n_gpus] > gpurun_out/measured_profile.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2507_10392_b200 import kernels
from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan import emulated as E
from paper_2507_10392_b200.runtime.model import (alloc_acts, alloc_bwd_scratch, init_flat,
                                                 layer_layout, make_model_ops)


def time_ms(fn, iters=10):
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


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2-small-124m"
    n_gpus = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg = E.MODELS[name]
    dev = torch.device("cuda", 0)
    lay = layer_layout(cfg)
    flat = init_flat(lay, "layer", 0, cfg, 1234).to(dev).bfloat16()
    gflat = torch.zeros(lay.numel, device=dev)
    p, g = lay.views(flat), lay.views(gflat)
    mo = make_model_ops(cfg, kernels)
    samples = []
    for b in (1, 2, 4, 8):
        n = b * cfg.seq_len
        acts = alloc_acts(cfg, n, dev)
        scr = alloc_bwd_scratch(cfg, n, dev)
        x = torch.randn(n, cfg.d_model, device=dev).bfloat16()
        out = torch.empty_like(x)
        dy = torch.randn(n, cfg.d_model, device=dev).bfloat16() * 0.01
        dx = torch.empty_like(x)
        f = time_ms(lambda: mo.layer_fwd(p, x, out, acts, n))
        bw = time_ms(lambda: mo.layer_bwd(p, g, x, dy, dx, acts, scr, n))
        samples.append([float(b), f * 1e-3, bw * 1e-3])
        print(f"# batch {b}: fwd {f:.3f} ms  bwd {bw:.3f} ms", file=sys.stderr)
    half = n_gpus // 2
    raw = E.profile_json([("n0", ["b200"] * (n_gpus - half) + ["b200h"] * half)])
    raw["runtime_samples"] = {
        "b200": {"transformer": samples},
        "b200h": {"transformer": [[b, 2 * f, 2 * bw] for b, f, bw in samples]},
    }
    prof = E.profile_from_json(raw)
    rt = P.fit_runtime_model(prof)
    gb = 8 * n_gpus
    plan, records = P.plan_training(prof, cfg.model_spec(), P.WorkloadSpec(gb, cfg.seq_len), rt,
                                    k_max=1)
    out = {"model": name, "cluster_profile": raw, "fits": {f"{k}/{c}": vars(v) for (k, c), v in rt.fits.items()},
           "plan": plan.to_json_dict(), "n_candidates": len(records)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
