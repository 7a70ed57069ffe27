"""Correctness of the NVLink peer collectives for a DP group of 8 ranks (the driver's
N=8 bench) on a box with fewer GPUs: ranks share GPUs round-robin (CUDA IPC works
between processes on one device), torch.distributed runs on gloo (NCCL refuses two
ranks per GPU).  Checks AllGather-v and the fused RS-v + AdamW kernel against torch
on the same uneven shard layout (config-2 shares 11x4 / 5x4), three steps.

    python -m torch.distributed.run --nproc-per-node 8 scripts/peer8_check.py
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2507_10392_b200.plan.shard import split_flat
from paper_2507_10392_b200.runtime.comm import PeerGroup
from paper_2507_10392_b200.runtime.executor import AdamConfig, Arena


class Unit:
    def __init__(self, arena, key, spec, pos, dev):
        self.full_off, self.grad_off, self.flag_off = arena.offsets[key]
        self.lo, self.hi = spec.bounds[pos]
        P = spec.bounds[-1][1]
        self.full = arena.view(self.full_off, P, torch.bfloat16)
        self.grad = arena.view(self.grad_off, P, torch.float32)
        m = self.hi - self.lo
        self.master = torch.zeros(m, device=dev)
        self.exp_avg = torch.zeros(m, device=dev)
        self.exp_avg_sq = torch.zeros(m, device=dev)
        self.counts, self.displs = spec.counts, spec.displs
        self.peer_cache = None


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    dev = torch.device("cuda", rank % ngpu)
    dist.init_process_group("gloo")
    shares = [11] * (world // 2) + [5] * (world - world // 2)
    P = 7087872 + 320  # GPT-2-small layer + a ragged tail
    spec = split_flat(P, shares)
    arena = Arena([("u", P)], dev)
    u = Unit(arena, "u", spec, rank, dev)
    peer = PeerGroup.build(dist, arena, rank, [list(range(world))])
    step = torch.zeros(1, device=dev, dtype=torch.int32)
    peer.epoch = step
    a = AdamConfig()
    g = torch.Generator().manual_seed(99)
    init = torch.randn(P, generator=g)
    u.master.copy_(init[u.lo:u.hi].to(dev))
    u.full.fill_(float("nan"))
    u.full[u.lo:u.hi] = u.master.to(torch.bfloat16)
    torch.cuda.synchronize()
    dist.barrier()
    ref = init.clone()
    m_ref, v_ref = torch.zeros(P), torch.zeros(P)
    ok = True
    worst = 0.0
    for t in range(1, 4):
        step.fill_(t)
        peer.allgather_unit(u)                      # every rank: full = all shards
        torch.cuda.synchronize()
        full = u.full.float().cpu()
        # bf16 of each rank's master; tiny fp32 differences vs torch may flip a rounding
        ag_ok = bool(torch.allclose(full, ref.to(torch.bfloat16).float(), rtol=1e-2, atol=1e-2))
        ag_ok &= bool(torch.isfinite(full).all())
        ok &= ag_ok
        grads = [torch.randn(P, generator=torch.Generator().manual_seed(1000 * t + r))
                 for r in range(world)]
        u.grad.copy_(grads[rank].to(dev))
        torch.cuda.synchronize()
        dist.barrier()
        sumsq = torch.zeros(1, device=dev)
        peer.reduce_scatter_adamw(u, a, sumsq, step, write_grad=True)
        torch.cuda.synchronize()
        gsum = torch.stack(grads).sum(0)
        got_g = u.grad[u.lo:u.hi].cpu()
        rs_ok = bool(torch.allclose(got_g, gsum[u.lo:u.hi], rtol=1e-5, atol=1e-4))
        ok &= rs_ok
        if not (ag_ok and rs_ok):
            print(json.dumps({"rank": rank, "step": t, "ag_ok": ag_ok, "rs_ok": rs_ok}), flush=True)
        # torch AdamW on the full vector, compared on this rank's shard
        bc1, bc2 = 1 - a.beta1 ** t, 1 - a.beta2 ** t
        ref.mul_(1 - a.lr * a.weight_decay)
        m_ref.mul_(a.beta1).add_(gsum, alpha=1 - a.beta1)
        v_ref.mul_(a.beta2).addcmul_(gsum, gsum, value=1 - a.beta2)
        ref.addcdiv_(m_ref, (v_ref.sqrt() / bc2 ** 0.5).add_(a.eps), value=-a.lr / bc1)
        err = (u.master.cpu() - ref[u.lo:u.hi]).abs().max().item()
        worst = max(worst, err)
        ok &= err < 1e-5
        dist.barrier()
    print(json.dumps({"rank": rank, "world": world, "gpu": rank % ngpu, "shard": [u.lo, u.hi],
                      "ok": ok, "max_master_err": worst}), flush=True)
    dist.barrier()
    peer.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
