"""Offline GEMM tile tuning for a workload (writes the committed, read-only tile
table paper_2507_10392_b200/gemm_tune_cache.txt; the library never writes it).

Runs one eager step of the workload with the GEMM front end wrapped, collects the
distinct call shapes, times the cost model's tile and its neighbours for each with
zb_gemm_tune (scratch outputs; inputs only read) and merges the winners into the
table, tagged with the current kernel generation ("g1").

  python scripts/tune_gemm.py [--gpus 1] [--append] [--seqs N]   (bench workload, GPT-2 small)
  --seqs: sequences on the tuning rank (default 8 = the N=1 bench); the N=2/4/8 layouts
  put 11 and 5 sequences on their ranks, so their shapes are tuned with --seqs 11 / 5.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
from paper_2507_10392_b200 import kernels as K
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

TABLE = os.path.join(ROOT, "paper_2507_10392_b200", "gemm_tune_cache.txt")
TAG = "g1"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--append", action="store_true", help="keep entries of other shapes")
    ap.add_argument("--out", default=TABLE, help="where to write the table")
    ap.add_argument("--seqs", type=int, default=8, help="sequences on the tuning rank")
    ap.add_argument("--model", default="gpt2-small-124m",
                    help="model whose per-rank GEMM shapes are tuned (plan/emulated.py MODELS)")
    ap.add_argument("--layers", type=int, default=0,
                    help="layers instantiated for tuning (every layer has the same shapes)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    import dataclasses
    from paper_2507_10392_b200.plan import emulated as E
    mcfg = E.MODELS[args.model]
    if args.layers:
        mcfg = dataclasses.replace(mcfg, n_layer=args.layers)
    cfg, plan, ctx, gb = bench.build_workload(args.gpus, per_gpu_batch=args.seqs, cfg=mcfg)
    if args.gpus != 1:
        raise SystemExit("single-process tuning: the per-rank shapes of rank 0 of an N-rank "
                         "layout are those of its share; run with --gpus 1 per share size")
    tr = ZorseTrainer(plan, ctx, cfg)
    calls = {}
    real = K.gemm

    def spy(a, b, out, **kw):
        M = a.shape[1] if kw.get("a_t") else a.shape[0]
        N = b.shape[1] if kw.get("b_t") else b.shape[0]
        Kd = a.shape[0] if kw.get("a_t") else a.shape[1]
        key = (M, N, Kd, int(kw.get("a_t", False)), int(kw.get("b_t", False)),
               kw.get("epilogue", 0), 1 if kw.get("beta", 0.0) == 1.0 else 0, out.stride(0))
        calls.setdefault(key, (a, b, out, dict(kw)))
        return real(a, b, out, **kw)

    K.gemm = spy
    tr.exec.model.ops.gemm = spy
    tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
    tr.exec.step()
    torch.cuda.synchronize()
    K.gemm = real
    rows = {}
    for key, (a, b, out, kw) in sorted(calls.items()):
        kw = {k: v for k, v in kw.items() if k in ("a_t", "b_t", "epilogue", "bias", "resid", "aux",
                                                   "beta")}
        if kw.get("epilogue") == K.EPI_BIAS_GELU:       # tune writes scratch outputs
            kw["aux"] = torch.empty_like(out)
        pair, bn, splits = K.gemm_tune(a, b, out, **kw)
        rows[key] = (pair, bn, splits)
        print(key, "->", rows[key], flush=True)
    old = []
    if args.append and os.path.exists(TABLE):
        for ln in open(TABLE):
            parts = ln.split()
            if len(parts) == 12 and parts[0] == TAG and tuple(map(int, parts[1:9])) not in rows:
                old.append(ln.rstrip("\n"))
    with open(args.out, "w") as fh:
        fh.write("# zorse B200 GEMM tile table (scripts/tune_gemm.py): tag M N K a_mn b_mn epi "
                 "beta1 ldc pair bn splits\n")
        for ln in old:
            fh.write(ln + "\n")
        for key, val in rows.items():
            fh.write(" ".join(map(str, (TAG,) + key + val)) + "\n")
    print(f"wrote {len(rows)} shapes (+{len(old)} kept) to {args.out}")


if __name__ == "__main__":
    main()
