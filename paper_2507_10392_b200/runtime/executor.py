"""Per-rank executor of a hetplan ``TrainingPlan`` on B200.

Each rank (one process per GPU) walks the global event order of the plan's
schedule (``plan.schedule``; the reference's simulate.py task graph) filtered
to its DP group, and turns every modelled task into real work:

  AllGather      -> uneven in-place AllGather-v of the layer's bf16 flat buffer
  Fwd            -> embedding (first stage) + transformer blocks + LM head,
                    loss and dlogits (last stage); stores layer-boundary
                    checkpoints for every microbatch
  P2PSend/Recv   -> many-to-many reshuffle of boundary activations / grads
                    between asymmetric groups, following the plan's routing
  Recompute      -> block forwards again, keeping the internals for Bwd
  Bwd            -> block backwards; fp32 weight grads accumulate per layer
  ReduceScatter  -> uneven in-place ReduceScatter-v (sum) of the fp32 grads
  OptimStep      -> fused AdamW on this rank's shard of the ministage's layers
                    (interleaved optimizer: right after that ministage's RS)
  OffloadAct / LoadAct -> with offload_acts (INTERLEAVED strategy): interior
                    layer-boundary checkpoints copied to pinned host memory after
                    Fwd and back before Recompute, on a host-copy stream, with a
                    2-microbatch device ring; otherwise no-ops (HBM-resident)
  FreeParams       -> no-op: gathered parameters stay resident in the arena

Every rank of every group issues its communication in one global order, so
the NCCL calls can never form the cyclic wait the paper had to work around
with Gloo.

Samples: microbatch m covers global samples [m*mbs, (m+1)*mbs); inside a group
they are dealt contiguously to devices in ``routing[group][m]`` order
(configure.py:414-430), so a boundary transfer is the set of interval
intersections between the sending and the receiving group's sample ranges.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from ..plan.configure import TrainingPlan
from ..plan.costs import CostContext
from ..plan.emulated import ModelConfig
from ..plan.schedule import Event, build_schedule
from ..plan.shard import ShardSpec, split_flat
from .transfers import boundary_transfers, sample_ranges
from .model import (FlatLayout, make_model_ops, alloc_acts, alloc_bwd_scratch, embed_layout,
                    head_layout, init_flat, layer_layout)


@dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1


class ParamUnit:
    """One flat parameter buffer (a layer, the embedding or the head) on one rank.

    full  : bf16 [P]  gathered parameters (this rank's shard lives in place at [lo, hi))
    grad  : fp32 [P]  gradient accumulator; after RS-v its [lo, hi) slice is the shard sum
    master, exp_avg, exp_avg_sq : fp32 [hi - lo]  optimizer state of the shard

    ``full`` and ``grad`` are views into the rank's arena (see ``Arena``) at byte
    offsets ``full_off`` / ``grad_off``; ``flag_off`` is the unit's 16-byte flag
    record there (used by the NVLink peer collectives).
    """

    def __init__(self, name: str, layout: FlatLayout, spec: ShardSpec, pos: int, init_full,
                 device, arena: "Arena", key):
        self.name, self.layout, self.spec, self.pos = name, layout, spec, pos
        self.lo, self.hi = spec.bounds[pos]
        n = self.hi - self.lo
        self.master = init_full[self.lo:self.hi].to(device=device, dtype=torch.float32).clone()
        self.exp_avg = torch.zeros(n, device=device, dtype=torch.float32)
        self.exp_avg_sq = torch.zeros(n, device=device, dtype=torch.float32)
        self.full_off, self.grad_off, self.flag_off = arena.offsets[key]
        self.full = arena.view(self.full_off, layout.numel, torch.bfloat16)
        self.full.fill_(float("nan"))
        self.full[self.lo:self.hi] = self.master.to(torch.bfloat16)
        self.grad = arena.view(self.grad_off, layout.numel, torch.float32)
        self.p = layout.views(self.full)
        self.g = layout.views(self.grad)
        self.counts = spec.counts
        self.displs = spec.displs
        self.peer_cache = None   # per-unit ctypes arrays of the peer collectives

    @property
    def shard_numel(self) -> int:
        return self.hi - self.lo


class Arena:
    """One allocation per rank holding every parameter unit's bf16 ``full`` buffer,
    then every fp32 ``grad`` buffer (contiguous, so one memset clears them), then a
    16-byte flag record per unit.  Every rank of a DP group holds the same units in
    the same order, so all offsets agree across the group — the NVLink peer
    collectives address a peer's buffer as (peer arena base + offset)."""

    ALIGN = 256

    def __init__(self, units: Sequence[Tuple[object, int]], device):
        a = self.ALIGN
        rnd = lambda x: (x + a - 1) // a * a  # noqa: E731
        off = 0
        full = {}
        for key, numel in units:
            full[key] = off
            off = rnd(off + 2 * numel)
        self.grad_lo = off
        grad = {}
        for key, numel in units:
            grad[key] = off
            off = rnd(off + 4 * numel)
        self.grad_hi = off
        self.flags_off = off
        off = rnd(off + 16 * len(units))
        self.nbytes = off
        self.offsets = {key: (full[key], grad[key], self.flags_off + 16 * i)
                        for i, (key, _) in enumerate(units)}
        self.buf = torch.empty(self.nbytes, device=device, dtype=torch.uint8)
        self.buf[self.flags_off:].zero_()

    def view(self, off: int, numel: int, dtype) -> torch.Tensor:
        nb = numel * torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + nb].view(dtype)

    def zero_grads(self) -> None:
        self.buf[self.grad_lo:self.grad_hi].view(torch.float32).zero_()


class StageExecutor:
    """Runs one rank's part of every training step of ``plan``."""

    def __init__(self, plan: TrainingPlan, ctx: CostContext, cfg: ModelConfig, dev_id: str,
                 rank_of: Dict[str, int], world_comm, group_comm, ops, device,
                 seed: int = 1234, adam: AdamConfig = AdamConfig(), init_device="cpu",
                 schedule: str = "gpipe", streams: bool = False, offload_acts: bool = False):
        if plan.routing is None:
            raise ValueError("plan has no routing; attach it (configure.attach_routing) first")
        if ctx.model.num_layers != cfg.n_layer:
            raise ValueError("model spec and model config disagree on the layer count")
        self.plan, self.ctx, self.cfg, self.dev_id = plan, ctx, cfg, dev_id
        self.rank_of = rank_of
        self.world, self.group_comm, self.ops, self.device = world_comm, group_comm, ops, device
        self.adam = adam
        self.model = make_model_ops(cfg, ops)
        self.schedule = build_schedule(ctx, plan, schedule)
        self.events: List[Event] = self.schedule.stream_for(dev_id)
        self.order = plan.global_order()
        self.ranges = plan.stage_layer_ranges()
        self.n_stages = len(self.order)
        self.gi = self.schedule.group_of_device(dev_id)
        self.group = plan.groups[self.gi]
        self.pos = self.group.device_ids.index(dev_id)
        self.share = self.group.shares[dev_id]
        S = cfg.seq_len
        self.n_tok = self.share * S
        self.mbs = plan.microbatch_size
        self.M = plan.n_microbatches
        self.global_tokens = ctx.workload.global_batch * S
        self.my_stages = [s for s in range(self.n_stages) if self.order[s][0] == self.gi]
        self.has_embed = self.order[0][0] == self.gi
        self.has_head = self.order[-1][0] == self.gi
        self.step_count = 0
        # Lanes -> CUDA streams: compute on the current stream, collectives and P2P on
        # their own streams, ordered by the task graph's dependencies (cross-stream
        # events), so gathers / reduce-scatters / transfers overlap compute.
        self.multistream = bool(streams) and device.type == "cuda"
        if self.multistream:
            self.lane_streams = {"collective": torch.cuda.Stream(device=device),
                                 "p2p": torch.cuda.Stream(device=device),
                                 "host": torch.cuda.Stream(device=device)}
        self.record_timeline = False  # measured Gantt (see measured_timeline)
        self._marks = []
        self.capture_grads = False   # tests: keep each reduced grad shard before Adam
        self.captured: Dict[object, torch.Tensor] = {}

        # ---------------- parameters (uneven ZeRO-3 shards) ----------------
        shares = [self.group.shares[d] for d in self.group.device_ids]
        self.units: Dict[object, ParamUnit] = {}
        lay = layer_layout(cfg)
        if lay.numel != ctx.model.params_of(0):
            raise ValueError(f"layer layout has {lay.numel} params, planner spec says "
                             f"{ctx.model.params_of(0)}")
        specs = []   # (key, layout, init kind, init index) in arena order
        for s in self.my_stages:
            for layer in range(*self.ranges[s]):
                specs.append((layer, lay, "layer", layer))
        if self.has_embed:
            specs.append(("embed", embed_layout(cfg), "embed", 0))
        if self.has_head:
            specs.append(("head", head_layout(cfg), "head", 0))
        self.arena = Arena([(k, l.numel) for k, l, _, _ in specs], device)
        for key, layout, kind, idx in specs:
            full = init_flat(layout, kind, idx, cfg, seed, device=init_device)
            name = f"layer{key}" if kind == "layer" else kind
            self.units[key] = ParamUnit(name, layout, split_flat(layout.numel, shares), self.pos,
                                        full, device, self.arena, key)
        # Group collectives: NCCL AG-v / RS-v + a separate AdamW launch, or a
        # communicator with ``fused_optimizer`` (NVLink peer memory: RS-v + scale +
        # AdamW + cast in one kernel at the ReduceScatter event; OptimStep is then
        # empty for this group).
        self._zeroed = set()

        # ---------------- activations ----------------
        d = cfg.d_model
        n = max(self.n_tok, 1)
        bf = dict(device=device, dtype=torch.bfloat16)
        self.act: Dict[Tuple[int, int], torch.Tensor] = {}
        self.gbuf: Dict[Tuple[int, int], torch.Tensor] = {}
        # Host offload of activation checkpoints (the reference's OffloadAct / LoadAct
        # tasks, simulate.py:369-376 / 451-467; memory model costs.py:596-600): with
        # the INTERLEAVED strategy the interior layer-boundary checkpoints of a
        # ministage (inputs of its 2nd..last layer) live on the device only in a
        # 2-microbatch ring — microbatch m uses slot m % 2 — and are copied to pinned
        # host memory after Fwd and back before Recompute on their own stream.
        # Stage-boundary checkpoints (P2P endpoints) stay resident.
        self.offload = bool(offload_acts) and plan.strategy.offloads
        self.host_act: Dict[Tuple[int, int], torch.Tensor] = {}
        self.interior: Dict[int, List[int]] = {}
        pin = device.type == "cuda"
        for s in self.my_stages:
            lo, hi = self.ranges[s]
            self.interior[s] = list(range(lo + 1, hi)) if self.offload else []
            for m in range(self.M):
                for layer in range(lo, hi + 1):
                    if (layer, m) in self.act:
                        continue
                    if layer in self.interior[s] and m >= 2:
                        self.act[(layer, m)] = self.act[(layer, m % 2)]   # ring slot
                    else:
                        self.act[(layer, m)] = torch.empty(n, d, **bf)
                    if layer in self.interior[s]:
                        self.host_act[(layer, m)] = torch.empty(n, d, dtype=torch.bfloat16,
                                                                pin_memory=pin)
                for key in ((lo, m), (hi, m)):
                    if key not in self.gbuf:
                        self.gbuf[key] = torch.empty(n, d, **bf)
        max_ms = max(self.ranges[s][1] - self.ranges[s][0] for s in self.my_stages)
        self.acts = [alloc_acts(cfg, self.n_tok, device) for _ in range(max_ms)]
        self.fwd_acts = alloc_acts(cfg, self.n_tok, device)
        self.fwd_out = torch.empty(n, d, **bf)
        self.bscr = alloc_bwd_scratch(cfg, self.n_tok, device)
        self.dy_pp = [torch.empty(n, d, **bf), torch.empty(n, d, **bf)]
        if self.has_head:
            self.logits = torch.empty(n, cfg.vocab, **bf)
            self.hf = torch.empty(n, d, **bf)
            self.hf_mean = torch.empty(n, device=device)
            self.hf_rstd = torch.empty(n, device=device)
            self.dhf = torch.empty(n, d, **bf)
        self.tokens = torch.zeros(self.M, n, device=device, dtype=torch.int32)
        self.labels = torch.zeros(self.M, n, device=device, dtype=torch.int32)
        self.loss_sum = torch.zeros(1, device=device, dtype=torch.float32)
        self.step_dev = torch.zeros(1, device=device, dtype=torch.int32)  # Adam t on the device
        self.gsumsq = torch.zeros(1, device=device, dtype=torch.float32)

        # ---------------- sample ranges and boundary transfer lists ----------
        self._sample_ranges = sample_ranges(plan)
        self.transfers = boundary_transfers(plan, self._sample_ranges, dev_id, rank_of, S)

    # ------------------------------------------------------------ geometry
    def my_samples(self, m: int) -> Tuple[int, int]:
        lo, hi = self._sample_ranges[self.gi][m][self.dev_id]
        return m * self.mbs + lo, m * self.mbs + hi

    # ------------------------------------------------------------ data
    def load_batch(self, batch: torch.Tensor) -> int:
        """Copy this rank's token / label slices of the global batch
        ([global_batch, S+1] int32, ideally pinned host memory) to the device.
        Returns the number of bytes copied host->device."""
        S = self.cfg.seq_len
        nbytes = 0
        if self.n_tok == 0 or not (self.has_embed or self.has_head):
            return 0
        for m in range(self.M):
            lo, hi = self.my_samples(m)
            rows = batch[lo:hi]
            if self.has_embed:
                self.tokens[m, :self.n_tok].copy_(rows[:, :S].reshape(-1), non_blocking=True)
                nbytes += self.n_tok * 4
            if self.has_head:
                self.labels[m, :self.n_tok].copy_(rows[:, 1:].reshape(-1), non_blocking=True)
                nbytes += self.n_tok * 4
        return nbytes

    # ------------------------------------------------------------ step
    def step(self) -> None:
        """One training iteration (data must be loaded).  Enqueues everything on
        the current stream; does not synchronise."""
        self.step_count += 1
        self.ops.step_increment(self.step_dev)
        self._zeroed = set()
        if not self._fused:
            self.arena.zero_grads()
        self.loss_sum.zero_()
        self.gsumsq.zero_()
        if not self.multistream:
            for ev in self.events:
                _DISPATCH[ev.kind](self, ev)
            return
        self._step_multistream()

    def _step_multistream(self) -> None:
        main = torch.cuda.current_stream(self.device)
        timed = self.record_timeline
        start = torch.cuda.Event(enable_timing=timed)
        start.record(main)
        self._marks = [("start", start)] if timed else []
        streams = {"compute": main, **self.lane_streams}
        for st in self.lane_streams.values():
            st.wait_event(start)                     # fork (also joins a graph capture)
        done: Dict[tuple, list] = {}                 # task key -> [(stream, event)]
        last = {}
        for ev in self.events:
            waits = []
            for dep in ev.deps:
                waits.extend(done.get(dep, ()))      # deps of other groups are remote
            noop = ("FreeParams", "P2PRecv") if self.offload else \
                ("OffloadAct", "LoadAct", "FreeParams", "P2PRecv")
            if ev.kind in noop or ev.lane not in streams:
                done[ev.key] = waits                 # no-op: completion = its deps'
                continue
            lane = "p2p" if ev.kind == "P2PSend" else ev.lane
            st = streams[lane]
            for dst, e in waits:
                if dst is not st:
                    st.wait_event(e)
            if timed:
                b0 = torch.cuda.Event(enable_timing=True)
                b0.record(st)
            with torch.cuda.stream(st):
                _DISPATCH[ev.kind](self, ev)
            e = torch.cuda.Event(enable_timing=timed)
            e.record(st)
            if timed:
                self._marks.append((ev, b0, e))
            done[ev.key] = [(st, e)]
            last[lane] = e
        for lane, e in last.items():                 # join
            if lane != "compute":
                main.wait_event(e)

    # ------------------------------------------------------------ handlers
    def _extras(self, stage: int, forward: bool, first_index: bool, last_index: bool):
        out = []
        if forward:
            if stage == 0 and self.has_embed and first_index:
                out.append("embed")
            if stage == self.n_stages - 1 and self.has_head and first_index:
                out.append("head")
        return out

    @property
    def _fused(self) -> bool:
        return getattr(self.group_comm, "fused_optimizer", False)

    def _on_allgather(self, ev: Event) -> None:
        key = ev.key
        s, i = key[1], key[2]
        units = [ev.layer] + self._extras(s, key[0] == "AGf", i == 0, False)
        if self.group_comm is None:
            return
        fused = self._fused
        for u in units:
            pu = self.units[u]
            if fused:
                self.group_comm.allgather_unit(pu)
                # A peer reads this rank's grad buffer until its fused RS+AdamW of the
                # previous step ends; the gather above waited for exactly that
                # (param_ready of every peer), so the buffer is free from here on.
                if u not in self._zeroed:
                    self._zeroed.add(u)
                    pu.grad.zero_()
            else:
                self.group_comm.allgather_v(pu.full, pu.counts, pu.displs)

    def _on_reduce_scatter(self, ev: Event) -> None:
        s, i = ev.key[1], ev.key[2]
        lo, hi = self.ranges[s]
        units = [ev.layer]
        if s == 0 and self.has_embed and i == hi - lo - 1:
            units.append("embed")
        if s == self.n_stages - 1 and self.has_head and i == 0:
            units.append("head")
        if self.group_comm is None:
            return
        if self._fused:
            a = self.adam
            for u in units:
                pu = self.units[u]
                self.group_comm.reduce_scatter_adamw(pu, a, self.gsumsq, self.step_dev,
                                                     write_grad=self.capture_grads)
                if self.capture_grads:
                    self.captured[u] = pu.grad[pu.lo:pu.hi].clone()
            return
        for u in units:
            pu = self.units[u]
            self.group_comm.reduce_scatter_v(pu.grad, pu.counts, pu.displs)

    def _on_optim(self, ev: Event) -> None:
        s = ev.key[1]
        units = list(range(*self.ranges[s]))
        if s == 0 and self.has_embed:
            units.append("embed")
        if s == self.n_stages - 1 and self.has_head:
            units.append("head")
        if self._fused:
            return   # done at each unit's ReduceScatter (fused RS-v + AdamW)
        a = self.adam
        for u in units:
            pu = self.units[u]
            if self.capture_grads:
                self.captured[u] = pu.grad[pu.lo:pu.hi].clone()
            self.ops.adamw_shard(pu.master, pu.exp_avg, pu.exp_avg_sq, pu.grad[pu.lo:pu.hi],
                                 pu.full[pu.lo:pu.hi], self.gsumsq, a.lr, a.beta1, a.beta2, a.eps,
                                 a.weight_decay, 1.0, self.step_dev)

    def _on_fwd(self, ev: Event) -> None:
        s, m = ev.key[1], ev.key[2]
        if self.n_tok == 0:
            return
        lo, hi = self.ranges[s]
        n = self.n_tok
        if s == 0:
            self.model.embed_fwd(self.units["embed"].p, self.tokens[m], self.act[(lo, m)], n)
        for layer in range(lo, hi):
            self.model.layer_fwd(self.units[layer].p, self.act[(layer, m)][:n],
                                 self.act[(layer + 1, m)][:n], self.fwd_acts, n)
        if s == self.n_stages - 1:
            hu = self.units["head"]
            self.model.head_fwd_bwd(hu.p, hu.g, self.act[(hi, m)][:n], self.labels[m],
                                    self.gbuf[(hi, m)][:n], self.logits, self.hf, self.hf_mean,
                                    self.hf_rstd, self.dhf, self.loss_sum,
                                    1.0 / self.global_tokens, n)

    def _on_recompute(self, ev: Event) -> None:
        s, m = ev.key[1], ev.key[2]
        if self.n_tok == 0:
            return
        lo, hi = self.ranges[s]
        n = self.n_tok
        for j, layer in enumerate(range(lo, hi)):
            self.model.layer_fwd(self.units[layer].p, self.act[(layer, m)][:n], self.fwd_out[:n],
                                 self.acts[j], n, need_out=False)

    def _on_bwd(self, ev: Event) -> None:
        s, m = ev.key[1], ev.key[2]
        if self.n_tok == 0:
            return
        lo, hi = self.ranges[s]
        n = self.n_tok
        dy = self.gbuf[(hi, m)][:n]
        for j in reversed(range(hi - lo)):
            layer = lo + j
            dx = self.gbuf[(lo, m)][:n] if j == 0 else self.dy_pp[j & 1][:n]
            u = self.units[layer]
            self.model.layer_bwd(u.p, u.g, self.act[(layer, m)][:n], dy, dx, self.acts[j],
                                 self.bscr, n)
            dy = dx
        if s == 0:
            self.model.embed_bwd(self.units["embed"].g, self.tokens[m], self.gbuf[(lo, m)][:n], n)

    def _on_send(self, ev: Event) -> None:
        """One global transfer: the sending group sends, the receiving group
        receives (see Schedule.stream_for)."""
        kind, b, m = ev.key
        direction = "f" if kind == "PSf" else "b"
        lst = self.transfers[(direction, b, m)]
        if ev.group == self.gi:  # sender
            # PSf: output of stage b; PSb: gradient of stage b+1's input
            buf = self.act[(self.ranges[b][1], m)] if kind == "PSf" else \
                self.gbuf[(self.ranges[b + 1][0], m)]
            self.world.p2p([(peer, buf[lo:hi], True) for peer, lo, hi, snd in lst if snd])
        else:                    # receiver
            buf = self.act[(self.ranges[b + 1][0], m)] if kind == "PSf" else \
                self.gbuf[(self.ranges[b][1], m)]
            self.world.p2p([(peer, buf[lo:hi], False) for peer, lo, hi, snd in lst if not snd])

    def _on_recv(self, ev: Event) -> None:
        return None  # data was received at the matching P2PSend event

    def _on_offload(self, ev: Event) -> None:
        """OffloadAct: interior checkpoints of (stage, microbatch) -> pinned host."""
        if not self.offload or self.n_tok == 0:
            return
        s, m = ev.key[1], ev.key[2]
        n = self.n_tok
        for layer in self.interior.get(s, ()):
            self.host_act[(layer, m)][:n].copy_(self.act[(layer, m)][:n], non_blocking=True)

    def _on_load(self, ev: Event) -> None:
        """LoadAct: pinned host -> the microbatch's device ring slot, before Recompute."""
        if not self.offload or self.n_tok == 0:
            return
        s, m = ev.key[1], ev.key[2]
        n = self.n_tok
        for layer in self.interior.get(s, ()):
            self.act[(layer, m)][:n].copy_(self.host_act[(layer, m)][:n], non_blocking=True)

    def _noop(self, ev: Event) -> None:
        return None

    def measured_timeline(self):
        """Events of the last recorded step with measured (start, end) seconds
        relative to the step start; call after torch.cuda.synchronize()."""
        if not self._marks:
            raise RuntimeError("set record_timeline = True (multi-stream executor) and run a step")
        t0 = self._marks[0][1]
        out = []
        for ev, b, e in self._marks[1:]:
            out.append((ev, t0.elapsed_time(b) * 1e-3, t0.elapsed_time(e) * 1e-3))
        return out

    # ------------------------------------------------------------ results
    def gather_master(self, unit) -> Tuple[int, int, torch.Tensor]:
        pu = self.units[unit]
        return pu.lo, pu.hi, pu.master


_DISPATCH = {
    "AllGather": StageExecutor._on_allgather,
    "ReduceScatter": StageExecutor._on_reduce_scatter,
    "OptimStep": StageExecutor._on_optim,
    "Fwd": StageExecutor._on_fwd,
    "Recompute": StageExecutor._on_recompute,
    "Bwd": StageExecutor._on_bwd,
    "P2PSend": StageExecutor._on_send,
    "P2PRecv": StageExecutor._on_recv,
    "OffloadAct": StageExecutor._on_offload,
    "LoadAct": StageExecutor._on_load,
    "FreeParams": StageExecutor._noop,
}
