"""Run a BASELINE.json config layout (scaled to the GPUs present) through the
product path for a few steps; report tokens/s and loss.  torchrun, 1 process/GPU.

  torchrun --nproc-per-node 4 scripts/config_run.py xl_1+3      (config 3 shape on 4 GPUs)
  torchrun --nproc-per-node 4 scripts/config_run.py llama7b_2x2 (config 4: 1F1B, seq 2048)
  torchrun --nproc-per-node 4 scripts/config_run.py llama13b_plan4 (config 5: planner layout)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan import emulated as E
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

RUNS = {
    # config 3: GPT-2 XL, asymmetric stages with uneven DP (3+5 on 8 GPUs -> 1+3 on 4)
    "xl_1+3": dict(cfg=E.GPT2_XL, nodes=[("n0", ["b200"]), ("n1", ["b200", "b200", "b200h"])],
                   groups=[["n0-0"], ["n1-0", "n1-1", "n1-2"]], gb=16, M=4, counts=[1, 1],
                   strategy="zorse", schedule="gpipe"),
    "xl_3+5": dict(cfg=E.GPT2_XL, nodes=E.CONFIG_NODES["xl-3+5"],
                   groups=[["n0-0", "n0-1", "n0-2"], [f"n1-{i}" for i in range(5)]], gb=64, M=8,
                   counts=[1, 1], strategy="zorse", schedule="gpipe"),
    # config 4: Llama-7B, 1F1B, 2-way ZeRO-3 DP per stage (4 stages x 2 on 8 GPUs -> 2 x 2 on 4)
    "llama7b_2x2": dict(cfg=E.LLAMA_7B, nodes=[("n0", ["b200", "b200"]), ("n1", ["b200", "b200"])],
                        groups=[["n0-0", "n0-1"], ["n1-0", "n1-1"]], gb=8, M=4, counts=[1, 1],
                        strategy="pp-zero3", schedule="1f1b"),
    "llama7b_4x2": dict(cfg=E.LLAMA_7B, nodes=E.CONFIG_NODES["llama7b-4x2"],
                        groups=[[f"n{i}-0", f"n{i}-1"] for i in range(4)], gb=32, M=8,
                        counts=[1, 1, 1, 1], strategy="pp-zero3", schedule="1f1b"),
    # config 5: Llama-13B, planner-chosen layout (plan_training) on an emulated-kinds node
    # (half full-speed b200, half half-speed b200h; 8 GPUs -> 4)
    "llama13b_plan4": dict(cfg=E.LLAMA_13B, nodes=[("n0", ["b200", "b200", "b200h", "b200h"])],
                           gb=16, planner=True, schedule="gpipe"),
}


def main():
    name = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    r = RUNS[name]
    cfg = r["cfg"]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prof = E.profile_from_json(E.profile_json(r["nodes"]))
    rt = P.fit_runtime_model(prof)
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                        workload=P.WorkloadSpec(r["gb"], cfg.seq_len))
    if r.get("planner"):   # the reference's full search picks stages, shares and M
        plan, _ = P.plan_training(prof, ctx.model, ctx.workload, rt)
        r["strategy"] = plan.strategy.value
    else:
        plan = P.build_plan(ctx, prof, P.make_partition(ctx.graph, r["groups"]), r["M"],
                            r["counts"], P.Strategy(r["strategy"]), P.cluster_fingerprint(prof),
                            "transformer")
    if plan.routing is None:
        P.attach_routing(plan, rt, "transformer")
    t0 = time.time()
    tr = ZorseTrainer(plan, ctx, cfg, world_rank=rank, world_size=world, schedule=r["schedule"],
                      init_device="cuda",
                      offload_acts=False if "--no-offload" in sys.argv else None)
    init_s = time.time() - t0
    init_peak = torch.cuda.max_memory_allocated() / 2**30
    torch.cuda.reset_peak_memory_stats()   # the steps' peak, without the one-off init
    batch = synthetic_batch(cfg.vocab, cfg.seq_len, r["gb"], 1, pin=True)
    losses = [tr.step(batch)]  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        tr.load(batch)
        tr.run()
    e.record()
    torch.cuda.synchronize()
    ms = torch.tensor([s.elapsed_time(e) / steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    losses.append(tr.loss_device().item())
    mem = torch.cuda.max_memory_allocated() / 2**30
    gmem = torch.tensor([mem], device="cuda")
    dist.all_reduce(gmem, op=dist.ReduceOp.MAX)
    # per-rank peak vs the plan's Eq.2 estimate (costs.py:538-607, restated bit-exact)
    est = P.memory_estimate(ctx, plan, tr.exec.gi, tr.dev_id)
    mine = {"dev": tr.dev_id, "share": tr.exec.share, "max_alloc_gib": mem,
            "init_peak_gib": init_peak,
            "executor": {k: (v / 2**30 if isinstance(v, int) and v > 1024 else v)
                         for k, v in tr.exec.memory_report().items()},
            "estimate_gib": {"params": est.m_params / 2**30, "grads": est.m_grads / 2**30,
                             "optim": est.m_optim / 2**30, "activations": est.m_activations / 2**30,
                             "total": est.m_total / 2**30}}
    per_rank = [None] * world
    dist.all_gather_object(per_rank, mine)
    if rank == 0:
        tok = r["gb"] * cfg.seq_len
        print(json.dumps({"offload_acts": tr.exec.offload,
            "run": name, "model": cfg.name, "n_gpus": world, "schedule": r["schedule"],
            "strategy": r["strategy"], "groups": [[g.device_ids, g.layers_assigned, g.shares]
                                                  for g in plan.groups],
            "n_microbatches": plan.n_microbatches, "global_batch": r["gb"], "seq_len": cfg.seq_len,
            "ms_per_step": ms.item(), "tokens_per_s": tok / (ms.item() * 1e-3),
            "model_tflops_per_gpu": cfg.flops_per_token() * tok / (ms.item() * 1e-3) / 1e12 / world,
            "loss_first_last": losses, "max_mem_gib": gmem.item(), "init_s": init_s,
            "memory_per_rank": per_rank}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
