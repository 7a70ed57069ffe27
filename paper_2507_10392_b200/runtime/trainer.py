"""Public entry point: execute a hetplan ``TrainingPlan`` on B200 GPUs.

    trainer = ZorseTrainer(plan, ctx, model_cfg)          # one process per GPU
    loss = trainer.step(batch)                              # batch: [B, S+1] int32 (host)

``plan`` is exactly what the reference planner emits (configure.py:118-304,
plan file docs/file_formats.md:99-129) plus its routing; ``ctx`` is the
reference's CostContext (cluster graph, runtime fits, model, workload) —
the same inputs ``simulate_plan(ctx, plan)`` takes (simulate.py:590).  World
rank r runs the r-th device of the cluster profile.
"""

from __future__ import annotations

from typing import Optional

import torch

from ..plan.configure import TrainingPlan
from ..plan.costs import CostContext
from ..plan.emulated import ModelConfig
from .executor import AdamConfig, StageExecutor


class ZorseTrainer:
    def __init__(self, plan: TrainingPlan, ctx: CostContext, cfg: ModelConfig, *,
                 world_rank: int = 0, world_size: int = 1, seed: int = 1234,
                 adam: AdamConfig = AdamConfig(), init_device: str = "cpu",
                 schedule: str = "gpipe", streams: bool = True,
                 offload_acts: Optional[bool] = None, recompute: str = "auto",
                 _ops=None, _comms=None, _device=None):
        devices = list(ctx.graph.vertices)
        if len(devices) != world_size:
            raise ValueError(f"cluster profile has {len(devices)} devices but world size is "
                             f"{world_size} (one process per GPU)")
        self.rank_of = {d: i for i, d in enumerate(devices)}
        self.dev_id = devices[world_rank]
        self.world_rank, self.world_size = world_rank, world_size
        groups_ranks = [[self.rank_of[d] for d in g.device_ids] for g in plan.groups]
        if _ops is None:
            # Product path: B200 kernels; DP-group collectives over NVLink peer memory,
            # stage-boundary P2P and the loss all-reduce over NCCL.  No CPU fallback.
            if not torch.cuda.is_available():
                raise RuntimeError("ZorseTrainer needs a CUDA (B200) device; there is no CPU path")
            from .. import kernels as ops
            device = torch.device("cuda", torch.cuda.current_device())
            if world_size > 1:
                import torch.distributed as dist
                from .comm import build_comms
                world, group = build_comms(dist, world_rank, world_size, groups_ranks)
            else:
                world, group = None, None
        else:  # test harness injection (tests/cpu_ops.py)
            ops = _ops
            device = _device or torch.device("cpu")
            world, group = _comms(groups_ranks) if _comms else (None, None)
        self.world_comm = world
        self.ops = ops
        self.device = device
        self.exec = StageExecutor(plan, ctx, cfg, self.dev_id, self.rank_of, world, group, ops,
                                  device, seed=seed, adam=adam, init_device=init_device,
                                  schedule=schedule, streams=streams, offload_acts=offload_acts,
                                  recompute=recompute)
        if _ops is None and world_size > 1:
            # AG-v / fused RS-v+AdamW over NVLink peer memory (csrc/peer.cu)
            from .comm import PeerGroup
            peer = PeerGroup.build(dist, self.exec.arena, world_rank, groups_ranks)
            if peer is not None:
                self.exec.group_comm = peer
        self.loss_buf = torch.zeros(1, device=device, dtype=torch.float32)

        self.graph = None
        self.launches_per_step = None   # kernel launches recorded in the captured step

    def capture(self) -> None:
        """Capture one whole training step (every kernel, collective and P2P of
        this rank) into a CUDA graph; ``run``/``step`` then replay it.  Must be
        called after at least one eager step (it warms every code path)."""
        if self.device.type != "cuda":
            raise RuntimeError("CUDA-graph capture needs the B200 path")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        counter = getattr(self.ops, "launch_count", None)
        before = counter() if counter else 0
        with torch.cuda.graph(g):
            self.exec.step()
        self.launches_per_step = (counter() - before) if counter else None
        self.exec.step_count -= 1   # capture recorded the step, it did not run it
        self.graph = g

    def load(self, batch: torch.Tensor) -> int:
        """Host->device copy of this rank's slices of the global batch."""
        return self.exec.load_batch(batch)

    def run(self) -> None:
        """Enqueue one training step (no host synchronisation)."""
        if self.graph is not None:
            self.exec.step_count += 1
            self.graph.replay()
        else:
            self.exec.step()

    def loss_device(self) -> torch.Tensor:
        """Global mean loss of the last step as a device scalar (all ranks)."""
        self.loss_buf.copy_(self.exec.loss_sum)
        if self.world_comm is not None:
            self.world_comm.allreduce_sum(self.loss_buf)
        return self.loss_buf / self.exec.global_tokens

    def step(self, batch: torch.Tensor) -> float:
        self.load(batch)
        self.run()
        return float(self.loss_device().item())
