"""Measured vs simulated iteration timeline.

Runs the bench workload (or --small) for a few steps with per-event CUDA-event
timing and writes, in the reference simulator's Gantt CSV format
(simulate.py:115-126: start,end,kind,group,stage,microbatch,layer,lane,devices):
  gpurun_out/gantt_simulated_rank<r>.csv   (the reference cost model's schedule)
  gpurun_out/gantt_measured_rank<r>.csv    (B200 CUDA-event times, same events)
and a JSON summary with per-kind measured totals and the simulated/measured
iteration time (the analogue of `hetplan report`, cli.py:234-285).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer


def write_gantt(path, rows):
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["start", "end", "kind", "group", "stage", "microbatch", "layer", "lane", "devices"])
        for ev, t0, t1 in rows:
            w.writerow([repr(t0), repr(t1), ev.kind, ev.group, ev.stage, ev.microbatch, ev.layer,
                        ev.lane, " ".join(ev.device_ids)])


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, plan, ctx, gb = bench.build_workload(world)
    tr = ZorseTrainer(plan, ctx, cfg, world_rank=rank, world_size=world)
    ex = tr.exec
    tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
    for _ in range(3):
        tr.run()
    ex.record_timeline = True
    tr.run()
    torch.cuda.synchronize()
    measured = ex.measured_timeline()
    ex.record_timeline = False
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    write_gantt(os.path.join(ROOT, "gpurun_out", f"gantt_measured_rank{rank}.csv"), measured)
    write_gantt(os.path.join(ROOT, "gpurun_out", f"gantt_simulated_rank{rank}.csv"),
                [(e, e.start, e.end) for e in ex.events])
    per_kind = {}
    for ev, t0, t1 in measured:
        per_kind[ev.kind] = per_kind.get(ev.kind, 0.0) + (t1 - t0)
    summary = {"rank": rank, "device": ex.dev_id, "events": len(measured),
               "measured_iteration_s": max(t1 for _, _, t1 in measured),
               "simulated_iteration_s": ex.schedule.iteration_time,
               "measured_busy_s_by_kind": per_kind}
    print(json.dumps(summary), flush=True)
    with open(os.path.join(ROOT, "gpurun_out", f"timeline_summary_rank{rank}.json"), "w") as fh:
        json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
