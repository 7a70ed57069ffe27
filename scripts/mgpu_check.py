"""Multi-GPU parity run (torchrun, one process per GPU): executes a small GPT
through the product path (NVLink peer AG-v / fused RS-v+AdamW, many-to-many P2P
over NCCL) for LAYOUT, gathers every rank's gradient / update / Adam-moment shards
to rank 0, assembles the units and compares them tensor by tensor with the CPU
fp32 oracle (oracle/parity.py).  Rank 0 prints one JSON line; exits 1 on failure.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/mgpu_check.py LAYOUT
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist

from oracle import parity
from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan import emulated as E
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

CFG = E.ModelConfig("mgpu-gpt", "gpt", n_layer=4, d_model=256, n_head=4, vocab=2048, seq_len=128)
LLAMA = E.ModelConfig("mgpu-llama", "llama", n_layer=4, d_model=512, n_head=4, vocab=4096,
                      seq_len=256, d_ff=1376)
XLW = E.ModelConfig("mgpu-xl-width", "gpt", n_layer=2, d_model=1600, n_head=25, vocab=4096,
                    seq_len=256)
LAYOUTS = {
    # name: (nodes, groups, n_microbatches, ministage counts, strategy, global batch)
    "dp2": ([("n0", ["b200", "b200h"])], [["n0-0", "n0-1"]], 2, [2], "zorse", 8),
    "dp2z3": ([("n0", ["b200", "b200h"])], [["n0-0", "n0-1"]], 2, [2], "pp-zero3", 8),
    "pp2": ([("n0", ["b200"]), ("n1", ["b200h"])], [["n0-0"], ["n1-0"]], 2, [2, 2], "zorse", 8),
    "pp1+3": ([("n0", ["b200"]), ("n1", ["b200", "b200h", "b200h"])],
              [["n0-0"], ["n1-0", "n1-1", "n1-2"]], 2, [1, 1], "zorse", 8),
    "dp4z3": ([("n0", ["b200", "b200", "b200h", "b200h"])], [[f"n0-{i}" for i in range(4)]], 2,
              [2], "pp-zero3", 12),
    "pp2x2": ([("n0", ["b200", "b200h"]), ("n1", ["b200", "b200"])],
              [["n0-0", "n0-1"], ["n1-0", "n1-1"]], 2, [2, 2], "zorse", 8),
    # Llama, 1F1B, 2 stages x 2-way ZeRO-3 DP (config 4 in miniature)
    "llama1f1b2x2": ([("n0", ["b200", "b200"]), ("n1", ["b200", "b200"])],
                     [["n0-0", "n0-1"], ["n1-0", "n1-1"]], 4, [1, 1], "pp-zero3", 8),
    # BASELINE config 1 exactly: tiny GPT (4 layers, d 256, seq 128, V 50304), the golden
    # `tiny` plan (tests/golden/plans.json): 2 asymmetric stages, uneven 2-rank ZeRO-3 group
    "cfg1_tiny": (E.CONFIG_NODES["tiny-2stage"], [["n0-0", "n0-1"], ["n1-0"]], 2, [1, 1], "zorse", 8),
    # GPT-2-XL widths, asymmetric 1 + 3 stages (config 3 in miniature)
    "xl1+3": ([("n0", ["b200"]), ("n1", ["b200", "b200", "b200h"])],
              [["n0-0"], ["n1-0", "n1-1", "n1-2"]], 4, [1, 1], "zorse", 8),
}
CFGS = {"llama1f1b2x2": LLAMA, "xl1+3": XLW, "cfg1_tiny": E.TINY_GPT}
SCHED = {"llama1f1b2x2": "1f1b"}


def main():
    name = sys.argv[1]
    nodes, groups, M, counts, strategy, gb = LAYOUTS[name]
    CFG = CFGS.get(name, globals()["CFG"])
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    prof = E.profile_from_json(E.profile_json(nodes))
    rt = P.fit_runtime_model(prof)
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=CFG.model_spec(),
                        workload=P.WorkloadSpec(gb, CFG.seq_len))
    plan = P.build_plan(ctx, prof, P.make_partition(ctx.graph, groups), M, counts,
                        P.Strategy(strategy), P.cluster_fingerprint(prof), "transformer")
    P.attach_routing(plan, rt, "transformer")
    if name == "cfg1_tiny":   # the very plan the reference emits for config 1 (golden bytes)
        with open(os.path.join(ROOT, "tests", "golden", "plans.json")) as fh:
            golden = next(c for c in json.load(fh) if c["name"] == "tiny")
        assert plan.dumps() == golden["plan_json"], "config-1 plan differs from the reference's"
    graph = os.environ.get("ZB_GRAPH", "1") == "1"   # script option: step 2 replays a graph
    tr = ZorseTrainer(plan, ctx, CFG, world_rank=rank, world_size=world,
                      schedule=SCHED.get(name, "gpipe"))
    tr.exec.capture_grads = True
    orc = parity.OracleRun(CFG) if rank == 0 else None
    records, losses = [], []
    for step in (1, 2):
        batch = synthetic_batch(CFG.vocab, CFG.seq_len, gb, step)
        if step == 2 and graph:
            tr.capture()      # step 2 replays a CUDA graph of the whole step
        before = parity.snapshot(tr.exec)
        loss = tr.step(batch.pin_memory())
        rec = parity.executor_step_record(tr.exec, loss, before)
        allrec = [None] * world if rank == 0 else None
        dist.gather_object(rec, allrec, dst=0)
        if rank == 0:
            pairs, recs = parity.check_step(CFG, orc, batch, step, allrec)
            losses += [(step, a, b) for a, b in pairs]
            records += recs
    ok = True
    if rank == 0:
        ok = all(parity.loss_ok(a, b, st) for st, a, b in losses) and not parity.failures(records)
        print(json.dumps({"layout": name, "graph": graph, "world": world, "ok": ok,
                          "loss_rel": max(abs(a - b) / abs(b) for _, a, b in losses),
                          **parity.worst(records),
                          "failures": parity.failures(records)[:4]}, default=str), flush=True)
    flag = [ok]
    dist.broadcast_object_list(flag, src=0)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flag[0] else 1)


if __name__ == "__main__":
    main()
