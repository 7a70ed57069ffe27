"""AllGather-v / ReduceScatter-v (+AdamW) of one uneven ZeRO-3 DP group:
NCCL (grouped per-root broadcast / reduce, then a separate AdamW launch) vs the
NVLink peer-memory path (copy-engine or SM-pull AllGather-v; fused RS-v + AdamW).

    torchrun --nproc-per-node N scripts/coll_bench.py

Prints one JSON line per (size, op, path) from rank 0: time per call (max over
ranks), bytes each rank receives over NVLink, and GB/s against the 770 GB/s
measured peer-copy bandwidth (B200_PROFILING.md).
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2507_10392_b200.plan.configure import proportional_split
from paper_2507_10392_b200.plan.shard import split_flat
from paper_2507_10392_b200.runtime.comm import NcclComm, PeerGroup, build_comms
from paper_2507_10392_b200.runtime.executor import AdamConfig, Arena

NVLINK_GBS = 770.0


class Unit:
    def __init__(self, arena, key, spec, pos, dev):
        self.full_off, self.grad_off, self.flag_off = arena.offsets[key]
        n = arena.offsets  # noqa
        self.spec = spec
        self.lo, self.hi = spec.bounds[pos]
        P = spec.bounds[-1][1]
        self.full = arena.view(self.full_off, P, torch.bfloat16)
        self.grad = arena.view(self.grad_off, P, torch.float32)
        self.full.normal_()
        self.grad.normal_()
        m = self.hi - self.lo
        self.master = torch.randn(m, device=dev)
        self.exp_avg = torch.zeros(m, device=dev)
        self.exp_avg_sq = torch.zeros(m, device=dev)
        self.counts, self.displs = spec.counts, spec.displs
        self.peer_cache = None


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / iters], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", device_id=dev)
    shares = [11 if i < (world + 1) // 2 else 5 for i in range(world)]   # config 2 skew
    ranks = list(range(world))
    _, nccl = build_comms(dist, rank, world, [ranks])
    sizes = {"gpt2s_layer": 7087872, "gpt2xl_layer": 30740800, "llama7b_layer": 202383360}
    arena = Arena([(k, v) for k, v in sizes.items()], dev)
    units = {k: Unit(arena, k, split_flat(v, shares), rank, dev) for k, v in sizes.items()}
    step = torch.ones(1, device=dev, dtype=torch.int32)
    peer_ce = PeerGroup.build(dist, arena, rank, [ranks], mode=0)
    peer_ce.epoch = step
    a = AdamConfig()
    for name, P in sizes.items():
        u = units[name]
        recv_bf16 = (P - (u.hi - u.lo)) * 2
        # max over ranks of the received bytes (the slowest rank sets the time)
        rb = torch.tensor([recv_bf16], device=dev, dtype=torch.float64)
        dist.all_reduce(rb, op=dist.ReduceOp.MAX)
        rb = rb.item()
        res = []
        t = timeit(lambda: nccl.allgather_v(u.full, u.counts, u.displs))
        res.append(("allgather_v", "nccl", t, rb))
        peer_ce.mode = 0
        t = timeit(lambda: peer_ce.allgather_unit(u))
        res.append(("allgather_v", "peer-ce", t, rb))
        peer_ce.mode = 1
        t = timeit(lambda: peer_ce.allgather_unit(u))
        res.append(("allgather_v", "peer-sm", t, rb))
        sumsq = torch.zeros(1, device=dev)

        def nccl_rs():
            nccl.reduce_scatter_v(u.grad, u.counts, u.displs)
            from paper_2507_10392_b200 import kernels as K
            K.adamw_shard(u.master, u.exp_avg, u.exp_avg_sq, u.grad[u.lo:u.hi],
                          u.full[u.lo:u.hi], sumsq, a.lr, a.beta1, a.beta2, a.eps,
                          a.weight_decay, 1.0, step)
        t = timeit(nccl_rs)
        res.append(("reduce_scatter_v+adamw", "nccl", t, rb * 2))
        t = timeit(lambda: peer_ce.reduce_scatter_adamw(u, a, sumsq, step))
        res.append(("reduce_scatter_v+adamw", "peer-fused", t, rb * 2))
        if rank == 0:
            for op, path, ms, b in res:
                print(json.dumps({"unit": name, "params": P, "world": world, "shares": shares,
                                  "op": op, "path": path, "ms": round(ms, 4),
                                  "nvlink_bytes_per_rank": int(b),
                                  "gbs": round(b / ms / 1e6, 1),
                                  "frac_of_770": round(b / ms / 1e6 / NVLINK_GBS, 3)}),
                      flush=True)
    dist.barrier()
    peer_ce.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
