"""`hetplan report` for a plan EXECUTED on B200 (cli.py:234-285).

For one workload — the bench layout (default) or a BASELINE config layout from
scripts/config_run.py (``--config NAME``) — prints and writes (profiles/ or --out):

  latency: the plan's Eq.1 estimate (costs.py total_iteration_latency), the
           simulated iteration (simulate.py list schedule) and the MEASURED
           device-timed iteration (CUDA events around a step, max over ranks);
  memory:  per device the Eq.2 estimate (memory_estimate), the simulator's replayed
           peak (simulate.py:660-696, restated bit-exact) and the MEASURED peak
           (torch.cuda.max_memory_allocated over the steps);
  files:   <tag>_gantt_simulated.csv / <tag>_gantt_measured.csv (per-event CUDA-event
           start / end, same columns, simulate.py:115-126) and
           <tag>_memory_simulated.csv (simulate.py:128-137).

  torchrun --nproc-per-node N scripts/report.py [--config NAME] [--profile measured.json]
           [--tag TAG] [--out DIR]

``--profile`` plans on a measured cluster profile (scripts/profile_layers.py output,
the reference's profile format docs/file_formats.md:7-36) with plan_training — the
planner loop closed on B200 measurements.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan.schedule import write_gantt_csv, write_memory_csv
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer


def build(args, world):
    if args.profile:
        from paper_2507_10392_b200.plan import emulated as E
        cfg = E.MODELS[args.model]
        with open(args.profile) as fh:
            raw = json.load(fh)
        prof = E.profile_from_json(raw.get("cluster_profile", raw))   # profile_layers.py output
        if len(prof.devices) != world:
            raise SystemExit(f"profile has {len(prof.devices)} devices, world is {world}")
        rt = P.fit_runtime_model(prof)
        gb = args.global_batch or 8 * world
        ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                            workload=P.WorkloadSpec(gb, cfg.seq_len))
        plan, _ = P.plan_training(prof, ctx.model, ctx.workload, rt, k_max=args.k_max)
        return cfg, plan, ctx, gb, "gpipe"
    if args.run:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import config_run as C
        r = C.RUNS[args.run]
        cfg = r["cfg"]
        from paper_2507_10392_b200.plan import emulated as E
        prof = E.profile_from_json(E.profile_json(r["nodes"]))
        rt = P.fit_runtime_model(prof)
        ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                            workload=P.WorkloadSpec(r["gb"], cfg.seq_len))
        if r.get("planner"):
            plan, _ = P.plan_training(prof, ctx.model, ctx.workload, rt)
        else:
            plan = P.build_plan(ctx, prof, P.make_partition(ctx.graph, r["groups"]), r["M"],
                                r["counts"], P.Strategy(r["strategy"]),
                                P.cluster_fingerprint(prof), "transformer")
        if plan.routing is None:
            P.attach_routing(plan, rt, "transformer")
        return cfg, plan, ctx, r["gb"], r["schedule"]
    import bench
    cfg, plan, ctx, gb = bench.build_workload(world)
    return cfg, plan, ctx, gb, "gpipe"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", dest="run", default=None)
    ap.add_argument("--profile", default=None)
    ap.add_argument("--model", default="gpt2-small-124m")
    ap.add_argument("--global-batch", type=int, default=0)
    ap.add_argument("--k-max", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--tag", default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles"))
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, plan, ctx, gb, schedule = build(args, world)
    tr = ZorseTrainer(plan, ctx, cfg, world_rank=rank, world_size=world, schedule=schedule,
                      init_device="cuda")
    ex = tr.exec
    tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
    torch.cuda.reset_peak_memory_stats()
    tr.run()                      # eager warm-up
    tr.capture()
    for _ in range(2):
        tr.run()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        tr.run()
    e.record()
    torch.cuda.synchronize()
    step_s = s.elapsed_time(e) / args.steps * 1e-3
    # one eager step with per-event CUDA events for the measured Gantt
    graph, tr.graph = tr.graph, None
    ex.record_timeline = True
    tr.run()
    torch.cuda.synchronize()
    measured = [(t0, t1, ev) for ev, t0, t1 in ex.measured_timeline()]
    ex.record_timeline = False
    tr.graph = graph
    peak = torch.cuda.max_memory_allocated()
    mine = {"dev": tr.dev_id, "step_s": step_s, "peak": peak,
            "rows": [(t0, t1, ev.kind, ev.group, ev.stage, ev.microbatch, ev.layer, ev.lane,
                      tuple(ev.device_ids)) for t0, t1, ev in measured]}
    allr = [mine]
    if dist is not None:
        allr = [None] * world
        dist.all_gather_object(allr, mine)
    if rank == 0:
        est = P.total_iteration_latency(ctx, plan)
        sched = ex.schedule
        peaks, traces = sched.memory(ctx)
        measured_s = max(r["step_s"] for r in allr)
        devices = {}
        for gi, group in enumerate(plan.groups):
            for dev in group.devices:
                m = P.memory_estimate(ctx, plan, gi, dev.id)
                meas = next(r["peak"] for r in allr if r["dev"] == dev.id)
                devices[dev.id] = {"estimated_bytes": m.m_total,
                                   "simulated_peak_bytes": peaks[dev.id]["total"],
                                   "measured_peak_bytes": meas,
                                   "budget_bytes": dev.mem_capacity * 0.9,
                                   "fits": m.m_total <= dev.mem_capacity * 0.9}
        tag = args.tag or (args.run or ("profile" if args.profile else "bench")) + f"_n{world}"
        os.makedirs(args.out, exist_ok=True)
        base = os.path.join(args.out, f"r02_report_{tag}")
        payload = {"latency": {"estimated_s": est.l_total,
                               "simulated_s": sched.iteration_time,
                               "measured_s": measured_s,
                               "estimate_over_simulated": est.l_total / sched.iteration_time,
                               "measured_over_simulated": measured_s / sched.iteration_time},
                   "memory": devices,
                   "collective_counts": {str(k): v for k, v in sched.collective_counts().items()},
                   "strategy": plan.strategy.value, "model": cfg.name, "global_batch": gb,
                   "plan": json.loads(plan.dumps()) if args.profile else None,
                   "files": [base + s for s in ("_gantt_simulated.csv", "_gantt_measured.csv",
                                               "_memory_simulated.csv")]}
        write_gantt_csv(base + "_gantt_simulated.csv", sched.gantt_rows())
        rows = sorted((r for rr in allr for r in rr["rows"]), key=lambda t: (t[0], t[2]))
        write_gantt_csv(base + "_gantt_measured.csv", rows)
        write_memory_csv(base + "_memory_simulated.csv", traces)
        with open(base + ".json", "w") as fh:
            json.dump(payload, fh, indent=1)
        lat = payload["latency"]
        print(f"latency: estimated {lat['estimated_s']:.6f} s, simulated {lat['simulated_s']:.6f} s, "
              f"measured {lat['measured_s']:.6f} s")
        for d in sorted(devices):
            v = devices[d]
            print(f"  {d}: est {v['estimated_bytes'] / 1e9:.2f} GB, sim peak "
                  f"{v['simulated_peak_bytes'] / 1e9:.2f} GB, measured peak "
                  f"{v['measured_peak_bytes'] / 1e9:.2f} GB, budget {v['budget_bytes'] / 1e9:.2f} GB")
        print(json.dumps({"report": base + ".json", **lat}), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
