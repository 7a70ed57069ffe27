"""In-step time per kernel kind for the bench workload (1 GPU).

Every call the executor makes into the kernel module is bracketed by CUDA events
(external events, so they survive CUDA-graph capture); one captured step is
replayed and the per-call durations are summed per kind (GEMMs keyed by shape and
epilogue).  Unlike an ncu launch list this measures the kernels warm, back to back,
inside the real step.

    python scripts/step_breakdown.py [--json out.json]
"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_10392_b200 import kernels
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

EPI = {0: "bf16", 1: "bias", 2: "bias+gelu", 3: "bias+resid", 4: "gelu'", 5: "f32+=", 6: "resid",
       7: "bias+gelu (no aux)"}


class Timed:
    def __init__(self, ops):
        self.ops = ops
        self.records = []

    def __getattr__(self, name):
        fn = getattr(self.ops, name)
        if not callable(fn) or name.startswith("_") or name in ("launch_count",
                                                                  "reset_launch_count"):
            return fn

        def wrapped(*a, **kw):
            key = name
            if name == "gemm":
                A, B = a[0], a[1]
                a_t, b_t = kw.get("a_t", False), kw.get("b_t", False)
                M = A.shape[1] if a_t else A.shape[0]
                K = A.shape[0] if a_t else A.shape[1]
                N = B.shape[1] if b_t else B.shape[0]
                key = f"gemm {M}x{N}x{K} {'T' if a_t else 'N'}{'T' if b_t else 'N'} " \
                      f"{EPI.get(kw.get('epilogue', 0))}"
            s = torch.cuda.Event(enable_timing=True, external=True)
            e = torch.cuda.Event(enable_timing=True, external=True)
            s.record()
            r = fn(*a, **kw)
            e.record()
            self.records.append((key, s, e))
            return r
        return wrapped


def _llama_workload():
    """Two Llama-7B layers (d 4096, f 11008, 32 heads x 128, seq 2048), 4 sequences."""
    from paper_2507_10392_b200 import plan as P
    from paper_2507_10392_b200.plan import emulated as E
    cfg = E.ModelConfig("llama7b-2L", "llama", 2, 4096, 32, 32000, 2048, d_ff=11008)
    prof = E.profile_from_json(E.profile_json(E.dp_group_nodes(1)))
    rt = P.fit_runtime_model(prof)
    gb = 4
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                        workload=P.WorkloadSpec(gb, cfg.seq_len))
    plan = P.build_plan(ctx, prof, P.make_partition(ctx.graph, [[d.id for d in prof.devices]]),
                        1, [cfg.n_layer], P.Strategy.INTERLEAVED, P.cluster_fingerprint(prof),
                        "transformer")
    P.attach_routing(plan, rt, "transformer")
    return cfg, plan, ctx, gb


def main():
    if os.environ.get("ZB_BREAKDOWN_MODEL") == "llama":
        cfg, plan, ctx, gb = _llama_workload()
    else:
        cfg, plan, ctx, gb = bench.build_workload(1)
    tr = ZorseTrainer(plan, ctx, cfg)
    ex = tr.exec
    tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
    for _ in range(3):
        tr.run()
    tr.capture()
    for _ in range(3):
        tr.run()
    torch.cuda.synchronize()
    s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        tr.run()
    e0.record()
    torch.cuda.synchronize()
    step_ms = s0.elapsed_time(e0) / 10

    t = Timed(kernels)
    ex.ops = t
    ex.model.ops = t
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ex.step()
    ex.ops = kernels
    ex.model.ops = kernels
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for key, s, e in t.records:
        tot[key] += s.elapsed_time(e)
        cnt[key] += 1
    covered = sum(tot.values())
    rows = [{"kind": k, "calls": cnt[k], "us": round(v * 1e3, 1),
             "share_of_step": round(v / step_ms, 4)} for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    out = {"step_ms": step_ms, "timed_ms": covered, "untimed_ms": step_ms - covered, "kinds": rows}
    for r in rows:
        print(f"{r['share_of_step'] * 100:6.2f}%  {r['us']:9.1f} us  n={r['calls']:3d}  {r['kind']}")
    print(f"step {step_ms:.3f} ms, timed kernels {covered:.3f} ms")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
