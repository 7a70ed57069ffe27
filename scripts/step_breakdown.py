"""In-step time of every kernel class of the N=1 bench step: the step is captured as a
CUDA graph with the weight-gradient lane serialised and CUDA events around EVERY kernel
call (bench.TimedOps does this for the GEMMs only), replayed, and the event durations
are summed per entry point.  HBM-bound classes also get GB/s from their algorithmic
bytes.  python scripts/step_breakdown.py [--out FILE]"""
import argparse
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402


class AllTimed:
    """Kernel-module proxy: every call bracketed by events on the current stream."""

    SKIP = {"reset_launch_count", "launch_count", "call"}

    def __init__(self, ops):
        self.ops, self.records = ops, []

    def __getattr__(self, name):
        f = getattr(self.ops, name)
        if not callable(f) or name in self.SKIP or name.startswith("_") or name.isupper():
            return f

        def timed(*a, **kw):
            s = torch.cuda.Event(enable_timing=True, external=True)
            e = torch.cuda.Event(enable_timing=True, external=True)
            s.record()
            r = f(*a, **kw)
            e.record()
            key = name
            if name == "gemm":
                key = "gemm epi%d" % kw.get("epilogue", 0)
            self.records.append((key, s, e))
            return r
        return timed


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from paper_2507_10392_b200 import kernels
    from paper_2507_10392_b200.runtime.data import synthetic_batch
    from paper_2507_10392_b200.runtime.trainer import ZorseTrainer
    torch.cuda.set_device(0)
    cfg, plan, ctx, gb = bench.build_workload(1)
    trainer = ZorseTrainer(plan, ctx, cfg, world_rank=0, world_size=1)
    ex = trainer.exec
    trainer.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
    for _ in range(3):
        trainer.run()
    torch.cuda.synchronize()
    # the real step (graph, lane on) for reference
    trainer.capture()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    trainer.run()
    s0.record()
    for _ in range(10):
        trainer.run()
    e0.record()
    torch.cuda.synchronize()
    step_ms = s0.elapsed_time(e0) / 10
    timed = AllTimed(kernels)
    ex.ops = timed
    ex.model.ops = timed
    wl = getattr(ex.model, "wlane", None)
    if wl is not None:
        wl.enabled = False
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ex.step()
    g.replay()
    torch.cuda.synchronize()
    timed_recs = list(timed.records)
    s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s1.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    serial_ms = s1.elapsed_time(e1)
    agg, cnt = defaultdict(float), defaultdict(int)
    for k, s, e in timed_recs:
        agg[k] += s.elapsed_time(e)
        cnt[k] += 1
    total = sum(agg.values())
    rows = sorted(agg.items(), key=lambda kv: -kv[1])
    out = {"step_ms_graph": step_ms, "serial_step_ms": serial_ms, "sum_kernel_ms": total,
           "classes": [{"op": k, "ms": v, "share_of_serial": v / serial_ms, "calls": cnt[k]}
                       for k, v in rows]}
    print(f"step (graph, lanes on) {step_ms:.3f} ms; serial step {serial_ms:.3f} ms; "
          f"sum of bracketed kernels {total:.3f} ms")
    for k, v in rows:
        print(f"  {k:28s} {v * 1e3:9.1f} us  {100 * v / serial_ms:5.1f}%  calls {cnt[k]}")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
