"""Per-rank executor of a hetplan ``TrainingPlan`` on B200.

Each rank (one process per GPU) walks the global event order of the plan's
schedule (``plan.schedule``; the reference's simulate.py task graph) filtered
to its DP group, and turns every modelled task into real work:

  AllGather      -> uneven AllGather-v of the layer's bf16 shards into a
                    parameter window slot (the ZeRO-3 materialised window)
  Fwd            -> embedding (first stage) + transformer blocks + LM head,
                    loss and dlogits (last stage); stores layer-boundary
                    checkpoints for every microbatch
  P2PSend/Recv   -> many-to-many reshuffle of boundary activations / grads
                    between asymmetric groups, following the plan's routing
  Recompute      -> folded into Bwd: each layer's internals are recomputed from
                    its checkpoint right before its backward (one layer's
                    recompute set is live, not a ministage's)
  Bwd            -> block backwards; fp32 weight grads accumulate per unit in a
                    gradient window slot
  ReduceScatter  -> uneven ReduceScatter-v (sum) of the fp32 grads fused with the
                    scale, AdamW on this rank's shard and the bf16 cast (the
                    interleaved optimizer runs right after the unit's RS; a
                    single-rank group runs AdamW on the whole unit there)
  OptimStep      -> nothing left to do (done at each unit's ReduceScatter)
  FreeParams     -> releases the ministage's parameter window slot (FREEf/FREEb,
                    simulate.py:387-392, :516-521)
  OffloadAct / LoadAct -> with offload_acts (INTERLEAVED strategy): interior
                    layer-boundary checkpoints copied to pinned host memory after
                    Fwd and back before the backward, on a host-copy stream, with a
                    2-microbatch device ring

Memory follows the plan's residency contract (costs.py:538-600; simulate.py
_initial_memory :565-588, z3_window_bytes :223-229):
  * persistent per unit: this rank's bf16 parameter shard and fp32 master /
    exp_avg / exp_avg_sq shards (the 1/g part);
  * parameters materialised in window slots: INTERLEAVED holds at most two
    ministages (current + prefetch, the FREEf/FREEb ring); PP_ZERO3 two LAYERS
    (gathered per microbatch, layer by layer inside Fwd / Bwd, prefetch depth 2);
    PP_ZERO2 the whole stage.  A single-rank group computes on its shard directly;
  * gradients: full fp32 units only while a ministage accumulates, in gradient
    window slots reused once the previous holder was reduce-scattered on every
    rank of the group.
Slot assignment is a deterministic dry run over the event stream (``WindowPlan``),
identical on every rank of a group, so peers address each other's gradient slots
at the same arena offsets.

Every rank of every group issues its NCCL operations in one global order, so
they can never form the cyclic wait the paper had to work around with Gloo
(PAPER.md:858-863).

Samples: microbatch m covers global samples [m*mbs, (m+1)*mbs); inside a group
they are dealt contiguously to devices in ``routing[group][m]`` order
(configure.py:414-430) — see runtime/transfers.py.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from ..plan.configure import TrainingPlan
from ..plan.costs import CostContext
from ..plan.emulated import ModelConfig
from ..plan.schedule import Event, build_schedule
from ..plan.shard import split_flat
from .model import (FlatLayout, alloc_acts, alloc_bwd_scratch, embed_layout, head_layout,
                    init_flat, layer_layout, make_model_ops)
from .transfers import boundary_transfers, sample_ranges

ALIGN = 256


def _rnd(x: int) -> int:
    return (x + ALIGN - 1) // ALIGN * ALIGN


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


@dataclass
class AdamConfig:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.95
    eps: float = 1e-8
    weight_decay: float = 0.1


class ParamUnit:
    """One flat parameter buffer (a layer, the embedding or the head) on one rank.

    Persistent (the rank's 1/g part):
      shard : bf16 [hi - lo]  parameter shard, in the rank's arena (peers gather it)
      master, exp_avg, exp_avg_sq : fp32 [hi - lo]  optimizer state
    Bound by the executor while materialised / accumulating:
      full, p : bf16 [P] gathered parameters (a window slot; the shard itself for a
                single-rank group) and its named views
      grad, g : fp32 [P] gradient accumulator (a gradient window slot at arena
                offset grad_off) and its named views
    """

    def __init__(self, name: str, layout: FlatLayout, bounds, pos: int, init_full, device):
        self.name, self.layout, self.pos = name, layout, pos
        self.bounds = bounds
        self.lo, self.hi = bounds[pos]
        self.counts = [hi - lo for lo, hi in bounds]
        self.displs = [lo for lo, _ in bounds]
        n = self.hi - self.lo
        self.master = init_full[self.lo:self.hi].to(device=device, dtype=torch.float32).clone()
        self.exp_avg = torch.zeros(n, device=device, dtype=torch.float32)
        self.exp_avg_sq = torch.zeros(n, device=device, dtype=torch.float32)
        self.shard: Optional[torch.Tensor] = None
        self.shard_offs: List[int] = []   # byte offset of every group rank's shard in its arena
        self.flag_off = 0
        self.full: Optional[torch.Tensor] = None
        self.p = None
        self.grad: Optional[torch.Tensor] = None
        self.g = None
        self.grad_off = 0
        self.peer_cache = None   # ctypes arrays of the peer collectives

    @property
    def numel(self) -> int:
        return self.layout.numel

    @property
    def shard_numel(self) -> int:
        return self.hi - self.lo

    def bind_full(self, t: torch.Tensor) -> None:
        self.full = t
        self.p = self.layout.views(t)

    def bind_grad(self, t: torch.Tensor, off: int) -> None:
        self.grad, self.grad_off = t, off
        self.g = self.layout.views(t)


class WindowPlan:
    """Deterministic window-slot assignment for one rank (identical on every rank of
    its group: it depends only on the group's events and unit sizes).

    Gradient slots: a ministage (chunk) acquires one at its first gradient write
    (the head's forward for the last stage, else its first Bwd) and releases it
    after its last ReduceScatter event; a chunk takes the least recently released
    slot free at that point of the event stream (so the previous holder's
    ReduceScatter was already issued), with at least two slots so a backward
    overlaps the previous ministage's reduce-scatter.  Parameter slots (group size > 1, gathers once per pass): acquired at
    the chunk's first AllGather of a pass, released at the pass's FreeParams
    (INTERLEAVED); PP_ZERO2 keeps one slot per chunk for the whole step (the stage
    stays materialised).  Every acquisition records the slot's previous holder, so
    the executor can wait for it: for gradients on every rank of the group (the
    fused reduce-scatter reads peers' slots), for parameters only locally."""

    def __init__(self, events: Sequence[Event], chunks: Dict[int, List[object]],
                 head_stage: Optional[int], gather_params: bool, per_layer: bool):
        self.grad_slot: Dict[int, int] = {}
        self.grad_prev: Dict[int, Tuple[Optional[int], bool]] = {}
        self.param_slot: Dict[Tuple[str, int], int] = {}
        self.param_prev: Dict[Tuple[str, int], Optional[Tuple[str, int]]] = {}
        frees = any(ev.kind == "FreeParams" for ev in events)
        # two gradient slots at least (when there are two ministages): a ministage's
        # backward then never waits for the previous one's reduce-scatter + AdamW
        min_grad_slots = min(2, len(chunks))
        last_rs = {}
        for idx, ev in enumerate(events):
            if ev.kind == "ReduceScatter":
                last_rs[ev.stage] = idx
        g_free: List[int] = []
        g_holder: Dict[int, int] = {}
        g_n = 0
        p_free: List[int] = []
        p_holder: Dict[int, Tuple[str, int]] = {}
        p_n = 0
        for idx, ev in enumerate(events):
            s = ev.stage
            if s not in chunks:
                continue
            first_grad = ev.kind == "Bwd" or (ev.kind == "Fwd" and s == head_stage)
            if first_grad and s not in self.grad_slot:
                if g_free and g_n >= min_grad_slots:
                    slot = g_free.pop(0)        # least recently released
                else:
                    slot, g_n = g_n, g_n + 1
                self.grad_slot[s] = slot
                self.grad_prev[s] = (g_holder.get(slot), True)
                g_holder[slot] = s
            if ev.kind == "ReduceScatter" and last_rs.get(s) == idx:
                g_free.append(self.grad_slot[s])
            if gather_params and not per_layer:
                if ev.kind == "AllGather" and ev.key[2] == 0:
                    key = ("f" if ev.key[0] == "AGf" or not frees else "b", s)
                    if key not in self.param_slot:
                        if p_free:
                            p_free.sort()
                            slot = p_free.pop(0)
                        else:
                            slot, p_n = p_n, p_n + 1
                        self.param_slot[key] = slot
                        self.param_prev[key] = p_holder.get(slot)
                        p_holder[slot] = key
                if ev.kind == "FreeParams":
                    key = ("f" if ev.key[0] == "FREEf" else "b", s)
                    if key in self.param_slot:
                        p_free.append(self.param_slot[key])
        # a slot's first holder in a step waits for its last holder of the previous step
        for s, (prev, _) in list(self.grad_prev.items()):
            if prev is None:
                self.grad_prev[s] = (g_holder[self.grad_slot[s]], False)
        self.n_grad_slots = g_n
        self.n_param_slots = p_n

    def param_key(self, fwd: bool, s: int) -> Tuple[str, int]:
        key = ("f" if fwd else "b", s)
        return key if key in self.param_slot else ("f", s)


class Arena:
    """One allocation per rank, exported to the DP group with a CUDA IPC handle:

      [flags: 16 B per unit][gradient window slots][this rank's bf16 shards]

    Flag and gradient-slot offsets are identical on every rank of the group; shard
    offsets differ (uneven shards) and are computed for every rank by ``layout``."""

    @staticmethod
    def layout(unit_keys, shard_counts: Dict[object, List[int]], n_grad_slots: int,
               grad_slot_bytes: int, rank: int):
        """(flag offsets, gradient region offset, shard offsets of ``rank``, bytes)."""
        flags = {k: 16 * i for i, k in enumerate(unit_keys)}
        off = _rnd(16 * len(unit_keys))
        grad_lo = off
        off += n_grad_slots * grad_slot_bytes
        shards = {}
        for k in unit_keys:
            shards[k] = off
            off = _rnd(off + 2 * shard_counts[k][rank])
        return flags, grad_lo, shards, off

    def __init__(self, nbytes: int, device):
        self.nbytes = nbytes
        self.buf = torch.zeros(nbytes, device=device, dtype=torch.uint8)

    def view(self, off: int, numel: int, dtype) -> torch.Tensor:
        nb = numel * torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + nb].view(dtype)


class StageExecutor:
    """Runs one rank's part of every training step of ``plan``."""

    def __init__(self, plan: TrainingPlan, ctx: CostContext, cfg: ModelConfig, dev_id: str,
                 rank_of: Dict[str, int], world_comm, group_comm, ops, device,
                 seed: int = 1234, adam: AdamConfig = AdamConfig(), init_device="cpu",
                 schedule: str = "gpipe", streams: bool = False,
                 offload_acts: Optional[bool] = None, recompute: str = "auto"):
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
        self.g_size = len(self.group.device_ids)
        self.share = self.group.shares[dev_id]
        S = cfg.seq_len
        self.n_tok = self.share * S
        self.mbs = plan.microbatch_size
        self.M = plan.n_microbatches
        self.global_tokens = ctx.workload.global_batch * S
        self.my_stages = [s for s in range(self.n_stages) if self.order[s][0] == self.gi]
        self.has_embed = self.order[0][0] == self.gi
        self.has_head = self.order[-1][0] == self.gi
        self.per_layer = plan.strategy.gathers_per_microbatch
        self.step_count = 0
        # Lanes -> CUDA streams: compute on the current stream, collectives and P2P on
        # their own streams, ordered by the task graph's dependencies (cross-stream
        # events), so gathers / reduce-scatters / transfers overlap compute.  PP_ZERO3
        # layer gathers get a stream of their own (issued from inside Fwd / Bwd).
        self.multistream = bool(streams) and device.type == "cuda"
        if self.multistream:
            self.lane_streams = {"collective": torch.cuda.Stream(device=device),
                                 "p2p": torch.cuda.Stream(device=device),
                                 "host": torch.cuda.Stream(device=device)}
            self.gather_stream = torch.cuda.Stream(device=device)
            self.prep_stream = torch.cuda.Stream(device=device)   # gradient-slot handover
            self.opt_stream = torch.cuda.Stream(device=device)    # early embedding update
        self.record_timeline = False  # measured Gantt (see measured_timeline)
        self._marks = []
        self.capture_grads = False   # tests: keep each reduced grad shard before Adam
        self.captured: Dict[object, torch.Tensor] = {}

        # ---------------- parameters: uneven ZeRO-3 shards + window slots --------
        shares = [self.group.shares[d] for d in self.group.device_ids]
        lay = layer_layout(cfg)
        if lay.numel != ctx.model.params_of(0):
            raise ValueError(f"layer layout has {lay.numel} params, planner spec says "
                             f"{ctx.model.params_of(0)}")
        specs = []   # (key, layout, init kind, init index) in arena order
        self.chunks: Dict[int, List[object]] = {}
        for s in self.my_stages:
            keys = list(range(*self.ranges[s]))
            for layer in keys:
                specs.append((layer, lay, "layer", layer))
            self.chunks[s] = keys
        if self.has_embed:
            specs.append(("embed", embed_layout(cfg), "embed", 0))
            self.chunks[0].append("embed")
        if self.has_head:
            specs.append(("head", head_layout(cfg), "head", 0))
            self.chunks[self.n_stages - 1].append("head")
        # Units are initialised one at a time (the full fp32 init of a unit is a
        # transient of one unit, never of the stage): shard bounds first, then the
        # window plan and the arena, then per unit master / shard from its init.
        self.units: Dict[object, ParamUnit] = {}
        bounds = {key: split_flat(layout.numel, shares).bounds for key, layout, _, _ in specs}
        self.win = WindowPlan(self.events, self.chunks,
                              self.n_stages - 1 if self.has_head else None, self.g_size > 1,
                              self.per_layer)
        unit_keys = [k for k, *_ in specs]
        shard_counts = {k: [hi - lo for lo, hi in bounds[k]] for k in unit_keys}
        numel = {key: layout.numel for key, layout, _, _ in specs}
        self.grad_slot_bytes = max(sum(_rnd(4 * numel[u]) for u in units)
                                   for units in self.chunks.values())
        self.arena_layouts = [Arena.layout(unit_keys, shard_counts, self.win.n_grad_slots,
                                           self.grad_slot_bytes, r) for r in range(self.g_size)]
        flags, self.grad_lo, shard_off, nbytes = self.arena_layouts[self.pos]
        self.arena = Arena(nbytes, device)
        for key, layout, kind, idx in specs:
            init = init_flat(layout, kind, idx, cfg, seed, device=init_device)
            name = f"layer{key}" if kind == "layer" else kind
            pu = ParamUnit(name, layout, bounds[key], self.pos, init, device)
            self.units[key] = pu
            pu.flag_off = flags[key]
            pu.shard_offs = [self.arena_layouts[r][2][key] for r in range(self.g_size)]
            pu.shard = self.arena.view(shard_off[key], pu.shard_numel, torch.bfloat16)
            pu.shard.copy_(init[pu.lo:pu.hi].to(device=device, dtype=torch.bfloat16))
            del init
            if self.g_size == 1:
                pu.bind_full(pu.shard)    # single-rank group: the shard is the unit
        self._grad_unit_off: Dict[object, int] = {}    # byte offset inside the chunk's slot
        self._param_unit_off: Dict[object, int] = {}   # element offset inside a param slot
        for s, units in self.chunks.items():
            goff = poff = 0
            for u in units:
                self._grad_unit_off[u] = goff
                self._param_unit_off[u] = poff
                goff += _rnd(4 * self.units[u].numel)
                poff += _rnd(2 * self.units[u].numel) // 2
        # parameter window slots (local: peers never read them)
        self.param_slots: List[torch.Tensor] = []
        self.layer_slots: List[torch.Tensor] = []
        self.extra_full: Dict[object, torch.Tensor] = {}
        if self.g_size > 1:
            if self.per_layer:
                # PP_ZERO3: two layer slots (current + prefetch); embedding / head keep a
                # resident full buffer (they are not planner layers)
                self.layer_slots = [torch.empty(lay.numel, device=device, dtype=torch.bfloat16)
                                    for _ in range(2)]
                for k in ("embed", "head"):
                    if k in self.units:
                        self.extra_full[k] = torch.empty(self.units[k].numel, device=device,
                                                         dtype=torch.bfloat16)
            else:
                slot_elems = max(sum(_rnd(2 * self.units[u].numel) // 2 for u in units)
                                 for units in self.chunks.values())
                self.param_slots = [torch.empty(slot_elems, device=device, dtype=torch.bfloat16)
                                    for _ in range(self.win.n_param_slots)]

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
        # host memory after Fwd and back before the backward on their own stream.
        # Stage-boundary checkpoints (P2P endpoints) stay resident.  Default: on
        # exactly when the plan's strategy offloads (the reference's memory model).
        if offload_acts is None:
            offload_acts = plan.strategy.offloads
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
        # Recompute policy.  The paper checkpoints every layer boundary and recomputes
        # the block internals in the backward to save memory; on a
        # 180 GB B200 the plan's memory budget usually leaves room to keep them:
        #   "full"      recompute every block internal from the checkpoint (the paper);
        #   "selective" keep the attention block's outputs (attention output + LSE,
        #               x_mid = x + proj(attn)) of every (layer, microbatch): the
        #               recompute skips the attention forward and the projection GEMM
        #               (selective activation recomputation, Korthikanti et al. 2022);
        #   "none"      keep the whole recompute set of every (layer, microbatch): the
        #               backward recomputes nothing;
        #   "auto"      "none" when it fits this device's memory budget (90% of the
        #               device, as memory_fits uses) after the allocations above, else
        #               "selective".
        # Numerics are identical either way (the recomputed values are bit-identical
        # to the forward's).
        if recompute not in ("auto", "none", "selective", "full"):
            raise ValueError(f"recompute must be auto|none|selective|full, not {recompute!r}")
        pairs = [(layer, m) for s in self.my_stages for layer in range(*self.ranges[s])
                 for m in range(self.M)]
        if recompute == "auto":
            recompute = "none"
            if device.type == "cuda" and self.n_tok > 0:
                probe = alloc_acts(cfg, self.n_tok, device)
                per = sum(t.numel() * t.element_size() for t in vars(probe).values())
                del probe
                budget = 0.9 * torch.cuda.get_device_properties(device).total_memory
                if torch.cuda.memory_allocated(device) + 3 * per + len(pairs) * per > budget:
                    recompute = "selective"
        self.recompute = recompute if self.n_tok > 0 else "full"
        self.kept: Dict[Tuple[int, int], tuple] = {}
        self.kept_acts: Dict[Tuple[int, int], object] = {}
        if self.recompute == "selective":
            seqs = max(self.n_tok // S, 1)
            for key in pairs:
                self.kept[key] = (torch.empty(n, d, **bf),
                                  torch.empty(seqs, cfg.n_head, S, device=device,
                                              dtype=torch.float32),
                                  torch.empty(n, d, **bf))
        elif self.recompute == "none":
            for key in pairs:
                self.kept_acts[key] = alloc_acts(cfg, self.n_tok, device)
        self.rc_acts = alloc_acts(cfg, self.n_tok, device)   # one layer's recompute set
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
            self.dhf32 = torch.empty(n, d, device=device, dtype=torch.float32)
        self.tokens = torch.zeros(self.M, n, device=device, dtype=torch.int32)
        # this rank's [share, S+1] row block of each microbatch, copied host->device in
        # one piece (a contiguous slice of the pinned batch: an asynchronous copy)
        self.batch_stage = torch.zeros(self.M, self.share, S + 1, device=device,
                                       dtype=torch.int32)
        self.labels = torch.zeros(self.M, n, device=device, dtype=torch.int32)
        self.loss_sum = torch.zeros(1, device=device, dtype=torch.float32)
        self._head_fresh = False   # the head's gradient slot awaits its first accumulation
        self.step_dev = torch.zeros(1, device=device, dtype=torch.int32)  # Adam t on the device
        self.gsumsq = torch.zeros(1, device=device, dtype=torch.float32)
        # Row-split token-embedding update (single-rank group owning the embedding): the
        # table's gradient is nonzero only in the rows of this step's tokens, so only those
        # rows are cleared before the embedding backward and updated after it; the other
        # rows get their (zero-gradient) AdamW step early, off the critical path.
        self.sparse_embed = self.has_embed and self.g_size == 1 and self.n_tok > 0
        if self.sparse_embed:
            self.embed_mark = torch.zeros(cfg.vocab, device=device, dtype=torch.int32)

        # ---------------- sample ranges and boundary transfer lists ----------
        self._sample_ranges = sample_ranges(plan)
        self.transfers = boundary_transfers(plan, self._sample_ranges, dev_id, rank_of, S)
        self._done: Dict[tuple, list] = {}

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
            stage = self.batch_stage[m, :hi - lo]
            if rows.is_contiguous():
                stage.copy_(rows, non_blocking=True)   # rows of the batch: contiguous
                nbytes += rows.numel() * rows.element_size()
            else:
                stage.copy_(rows.contiguous(), non_blocking=True)
                nbytes += rows.numel() * 4
            n = (hi - lo) * S
            if self.has_embed:
                self.tokens[m, :n].view(hi - lo, S).copy_(stage[:, :S])
            if self.has_head:
                self.labels[m, :n].view(hi - lo, S).copy_(stage[:, 1:])
        return nbytes

    # ------------------------------------------------------------ memory report
    def memory_report(self) -> Dict[str, float]:
        """Bytes this rank allocates per category of the reference's memory model
        (costs.py:538-600): parameters (persistent bf16 shard + materialised window),
        gradients (fp32 window slots), optimizer (fp32 master/m/v shards),
        checkpoints (layer-boundary activations resident on the device)."""
        shard_bf16 = sum(2 * pu.shard_numel for pu in self.units.values())
        window = sum(t.numel() * 2 for t in self.param_slots + self.layer_slots)
        window += sum(t.numel() * 2 for t in self.extra_full.values())
        acts = {id(t): t.numel() * t.element_size() for t in self.act.values()}
        return {"params_shard": shard_bf16, "params_window": window,
                "grads_window": self.win.n_grad_slots * self.grad_slot_bytes,
                "optim": sum(12 * pu.shard_numel for pu in self.units.values()),
                "checkpoints": sum(acts.values()),
                "kept_activations": sum(a.numel() * 2 + b.numel() * 4 + c.numel() * 2
                                        for a, b, c in self.kept.values()) +
                sum(t.numel() * t.element_size() for acts in self.kept_acts.values()
                    for t in vars(acts).values()),
                "recompute": self.recompute,
                "grad_slots": self.win.n_grad_slots,
                "param_slots": len(self.param_slots) or len(self.layer_slots)}

    # ------------------------------------------------------------ step
    def step(self) -> None:
        """One training iteration (data must be loaded).  Enqueues everything on
        the current stream; does not synchronise."""
        self.step_count += 1
        self.ops.step_increment(self.step_dev)
        self.ops.fill_f32(self.loss_sum, 0.0)
        self.ops.fill_f32(self.gsumsq, 0.0)
        self._done = {}
        if self.sparse_embed:
            self.ops.embed_mark(self.tokens, self.cfg.vocab, self.embed_mark, self.step_dev)
        if not self.multistream:
            if self.sparse_embed:
                self._embed_update(marked=False)
            for ev in self.events:
                _DISPATCH[ev.kind](self, ev)
            return
        self._step_multistream()

    def _wte(self, t: torch.Tensor) -> torch.Tensor:
        """The token-embedding table's [V, d] view of an embed-unit flat buffer."""
        return t[:self.cfg.vocab * self.cfg.d_model].view(self.cfg.vocab, self.cfg.d_model)

    def _embed_update(self, marked: bool) -> None:
        """AdamW over the token-embedding rows this step's tokens touched (marked, after
        the backward) or did not touch (g = 0; any time in the step)."""
        pu, a = self.units["embed"], self.adam
        self.ops.adamw_rows(self._wte(pu.master), self._wte(pu.exp_avg), self._wte(pu.exp_avg_sq),
                            self._wte(pu.grad) if marked else None, self._wte(pu.shard),
                            self.gsumsq, self.embed_mark, marked, a.lr, a.beta1, a.beta2,
                            a.eps, a.weight_decay, 1.0, self.step_dev)

    def _step_multistream(self) -> None:
        main = torch.cuda.current_stream(self.device)
        timed = self.record_timeline
        start = torch.cuda.Event(enable_timing=timed)
        start.record(main)
        self._marks = [("start", start)] if timed else []
        streams = {"compute": main, **self.lane_streams}
        for st in list(self.lane_streams.values()) + [self.gather_stream, self.prep_stream,
                                                      self.opt_stream]:
            st.wait_event(start)                     # fork (also joins a graph capture)
        if self.sparse_embed and not self.has_head:  # (with the head: see _on_fwd)
            with torch.cuda.stream(self.opt_stream):
                self._embed_update(marked=False)

        done = self._done                            # task key -> [(stream, event)]
        last = {}
        noop = ("P2PRecv", "Recompute", "OptimStep", "FreeParams")
        if not self.offload:
            noop += ("OffloadAct", "LoadAct")
        for ev in self.events:
            waits = []
            for dep in ev.deps:
                waits.extend(done.get(dep, ()))      # deps of other groups are remote
            if ev.kind in noop or ev.lane not in streams or \
                    (ev.kind == "AllGather" and self._deferred_gather()):
                done[ev.key] = waits                 # marker: completion = its deps'
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
        for st in (self.gather_stream, self.prep_stream, self.opt_stream):
            j = torch.cuda.Event()
            j.record(st)
            main.wait_event(j)
        for lane, e in last.items():                 # join
            if lane != "compute":
                main.wait_event(e)

    def _wait_done(self, keys, stream=None) -> None:
        """Make the current (or the given) stream wait for the completion of task keys."""
        if not self.multistream:
            return
        st = stream or torch.cuda.current_stream(self.device)
        for k in keys:
            for src, e in self._done.get(k, ()):
                if src is not st:
                    st.wait_event(e)

    # ------------------------------------------------------------ windows
    def _deferred_gather(self) -> bool:
        """PP_ZERO3 with a DP group: gathers are issued layer by layer inside Fwd / Bwd."""
        return self.per_layer and self.g_size > 1

    def _skip_gathers(self) -> bool:
        """A zero-share rank computes nothing; with one-sided (peer-pull) gathers it
        need not gather either (peers only read its shard)."""
        return self.n_tok == 0 and getattr(self.group_comm, "one_sided", False)

    def _acquire_grads(self, s: int) -> None:
        """Bind the chunk's units to their gradient slot and clear it, once the slot's
        previous holder was reduce-scattered here and read by every peer.  The
        handover (peer waits + clearing) runs on its own stream, which depends only
        on the previous holder's ReduceScatter, so it is off the compute path."""
        units = self.chunks[s]
        if self.units[units[0]].grad is not None:
            return
        base = self.grad_lo + self.win.grad_slot[s] * self.grad_slot_bytes
        region = self.arena.view(base, self.grad_slot_bytes // 4, torch.float32)
        last = units[-1]
        used = self._grad_unit_off[last] // 4 + self.units[last].numel
        if last == "head" and self.n_tok > 0:
            # head_w (the head unit's last entry) is written by the LM-head wgrad GEMM with
            # beta = 0 on the slot's first accumulation (_on_fwd): no clearing needed
            hw_off = dict((n, o) for n, o, _ in self.units[last].layout.entries)["head_w"]
            used = self._grad_unit_off[last] // 4 + hw_off
            self._head_fresh = True
        prev, same_step = self.win.grad_prev[s]
        ps = self.prep_stream if self.multistream else None
        if prev is not None and same_step:
            n_rs = self.ranges[prev][1] - self.ranges[prev][0]
            self._wait_done([("RS", prev, i) for i in range(n_rs)], ps)
        with torch.cuda.stream(ps) if ps is not None else _nullctx():
            if prev is not None and self.group_comm is not None:
                for u in self.chunks[prev]:
                    self.group_comm.wait_consumed(self.units[u], 0 if same_step else -1,
                                                  self.step_dev)
            if self.sparse_embed and "embed" in units and not self.capture_grads:
                # only the rows of this step's tokens of the token-embedding gradient
                lo_e = self._grad_unit_off["embed"] // 4
                hi_e = lo_e + self.cfg.vocab * self.cfg.d_model
                self.ops.fill_f32(region[:lo_e], 0.0)
                self.ops.fill_f32(region[hi_e:used], 0.0)
                self.ops.embed_zero_rows(self.tokens, region[lo_e:hi_e].view(self.cfg.vocab,
                                                                              self.cfg.d_model))
            else:
                self.ops.fill_f32(region[:used], 0.0)
        if ps is not None:
            e = torch.cuda.Event()
            e.record(ps)
            torch.cuda.current_stream(self.device).wait_event(e)
        for u in units:
            pu = self.units[u]
            off = self._grad_unit_off[u]
            pu.bind_grad(region[off // 4:off // 4 + pu.numel], base + off)

    def _release_grads(self, s: int) -> None:
        for u in self.chunks[s]:
            pu = self.units[u]
            pu.grad, pu.g = None, None

    def _gather_unit(self, pu: ParamUnit, dst: torch.Tensor) -> None:
        """AllGather-v of one unit into ``dst`` (full [P] bf16), bound as its params."""
        pu.bind_full(dst)
        self.group_comm.gather(pu, dst, self.step_dev)

    # ------------------------------------------------------------ handlers
    def _extras(self, stage: int, forward: bool, first_index: bool):
        out = []
        if forward and first_index:
            if stage == 0 and self.has_embed:
                out.append("embed")
            if stage == self.n_stages - 1 and self.has_head:
                out.append("head")
        return out

    def _on_allgather(self, ev: Event) -> None:
        """Ministage window (INTERLEAVED / PP_ZERO2): gather the layer (and, at the
        first layer of a forward pass, the embedding / head) into the chunk's slot.
        A zero-share rank computes nothing and gathers nothing (it is only read)."""
        if self.group_comm is None or self._deferred_gather() or self._skip_gathers():
            return
        s, i = ev.key[1], ev.key[2]
        fwd = ev.key[0] == "AGf"
        wkey = self.win.param_key(fwd, s)
        if i == 0:
            prev = self.win.param_prev.get(wkey)
            if prev is not None:    # the slot's previous holder released it (FreeParams)
                self._wait_done([("FREE" + prev[0], prev[1])])
        region = self.param_slots[self.win.param_slot[wkey]]
        for u in [ev.layer] + self._extras(s, fwd, i == 0):
            pu = self.units[u]
            off = self._param_unit_off[u]
            self._gather_unit(pu, region[off:off + pu.numel])

    def _on_reduce_scatter(self, ev: Event) -> None:
        """RS-v + scale + AdamW + bf16 shard (fused kernel for a DP group; AdamW on the
        whole unit for a single-rank group); the chunk's gradient slot is released
        after its last ReduceScatter."""
        s, i = ev.key[1], ev.key[2]
        lo, hi = self.ranges[s]
        units = [ev.layer]
        if s == 0 and self.has_embed and i == hi - lo - 1:
            units.append("embed")
        if s == self.n_stages - 1 and self.has_head and i == 0:
            units.append("head")
        a = self.adam
        for u in units:
            pu = self.units[u]
            if self.group_comm is not None:
                self.group_comm.reduce_scatter_adamw(pu, a, self.gsumsq, self.step_dev,
                                                     write_grad=self.capture_grads)
            elif u == "embed" and self.sparse_embed:
                # token rows of this step (the others were updated early in the step),
                # then the rest of the unit (position embeddings) densely
                self._embed_update(marked=True)
                k = self.cfg.vocab * self.cfg.d_model
                if pu.numel > k:
                    self.ops.adamw_shard(pu.master[k:], pu.exp_avg[k:], pu.exp_avg_sq[k:],
                                         pu.grad[k:], pu.shard[k:], self.gsumsq, a.lr, a.beta1,
                                         a.beta2, a.eps, a.weight_decay, 1.0, self.step_dev)
            else:
                self.ops.adamw_shard(pu.master, pu.exp_avg, pu.exp_avg_sq, pu.grad, pu.shard,
                                     self.gsumsq, a.lr, a.beta1, a.beta2, a.eps,
                                     a.weight_decay, 1.0, self.step_dev)
            if self.capture_grads:
                self.captured[u] = pu.grad[pu.lo:pu.hi].clone()
        if i == hi - lo - 1:
            self._release_grads(s)

    def _on_fwd(self, ev: Event) -> None:
        s, m = ev.key[1], ev.key[2]
        if s == self.n_stages - 1 and self.has_head:
            self._acquire_grads(s)    # the head's backward runs inside the last Fwd
        if self._deferred_gather() and not self._skip_gathers():
            for u in self._extras(s, True, True):
                self._gather_unit(self.units[u], self.extra_full[u])
        lo, hi = self.ranges[s]
        if self.n_tok == 0:
            if self._deferred_gather() and not self._skip_gathers():
                self._layers(list(range(lo, hi)), lambda layer: None)
            return
        n = self.n_tok
        if s == 0:
            self.model.embed_fwd(self.units["embed"].p, self.tokens[m], self.act[(lo, m)], n)

        def body(layer):
            a = self.fwd_acts
            if self.recompute == "selective":
                attn, lse, x_mid = self.kept[(layer, m)]
                a = dataclasses.replace(a, attn=attn, lse=lse, x_mid=x_mid)
            elif self.recompute == "none":
                a = self.kept_acts[(layer, m)]
            self.model.layer_fwd(self.units[layer].p, self.act[(layer, m)][:n],
                                 self.act[(layer + 1, m)][:n], a, n,
                                 keep_preact=self.recompute == "none")
        self._layers(list(range(lo, hi)), body)
        if s == self.n_stages - 1:
            if self.sparse_embed and self.multistream and m == 0:
                # the untouched embedding rows' update (HBM-bound) overlaps the LM head's
                # compute-bound GEMMs (opt_stream is joined at the end of the step)
                self.opt_stream.wait_stream(torch.cuda.current_stream(self.device))
                with torch.cuda.stream(self.opt_stream):
                    self._embed_update(marked=False)
            hu = self.units["head"]
            self.model.head_fwd_bwd(hu.p, hu.g, self.act[(hi, m)][:n], self.labels[m],
                                    self.gbuf[(hi, m)][:n], self.logits, self.hf, self.hf_mean,
                                    self.hf_rstd, self.dhf, self.loss_sum,
                                    1.0 / self.global_tokens, n, dhf32=self.dhf32,
                                    first=self._head_fresh)
            self._head_fresh = False

    def _on_bwd(self, ev: Event) -> None:
        """Recompute + backward, layer by layer in reverse (each layer's internals are
        recomputed from its checkpoint right before its backward)."""
        s, m = ev.key[1], ev.key[2]
        self._acquire_grads(s)
        lo, hi = self.ranges[s]
        if self.n_tok == 0:
            if self._deferred_gather() and not self._skip_gathers():
                self._layers(list(reversed(range(lo, hi))), lambda layer: None)
            return
        n = self.n_tok
        state = {"dy": self.gbuf[(hi, m)][:n]}

        def body(layer):
            j = layer - lo
            dx = self.gbuf[(lo, m)][:n] if j == 0 else self.dy_pp[j & 1][:n]
            u = self.units[layer]
            x = self.act[(layer, m)][:n]
            if self.recompute == "none":
                a = self.kept_acts[(layer, m)]
            else:
                a = self.rc_acts
                if self.recompute == "selective":
                    attn, lse, x_mid = self.kept[(layer, m)]
                    a = dataclasses.replace(a, attn=attn, lse=lse, x_mid=x_mid)
                self.model.layer_fwd(u.p, x, self.fwd_out[:n], a, n, need_out=False,
                                     kept=self.recompute == "selective")
            self.model.layer_bwd(u.p, u.g, x, state["dy"], dx, a, self.bscr, n)
            state["dy"] = dx
        self._layers(list(reversed(range(lo, hi))), body)
        if s == 0:
            self.model.embed_bwd(self.units["embed"].g, self.tokens[m], self.gbuf[(lo, m)][:n], n)

    def _layers(self, layers: List[int], body) -> None:
        """Run ``body(layer)`` over a chunk's layers.  PP_ZERO3 with a DP group: each
        layer is gathered into one of two layer slots on the gather stream just in
        time (prefetch depth 2) and a slot is reused once the compute that read it is
        done — the two-layer materialised window of z3_window_bytes (simulate.py:
        223-229)."""
        if not self._deferred_gather():
            for layer in layers:
                body(layer)
            return
        if not self.multistream:
            for k, layer in enumerate(layers):
                self._gather_unit(self.units[layer], self.layer_slots[k % 2])
                body(layer)
            return
        comp = torch.cuda.current_stream(self.device)
        gs = self.gather_stream
        ag_done, use_done = {}, {}

        def gather(k):
            if k >= 2:
                gs.wait_event(use_done[k - 2])
            with torch.cuda.stream(gs):
                self._gather_unit(self.units[layers[k]], self.layer_slots[k % 2])
            e = torch.cuda.Event()
            e.record(gs)
            ag_done[k] = e

        gs.wait_stream(comp)     # the slots were last read by this stream's earlier work
        for k in range(min(2, len(layers))):
            gather(k)
        for k, layer in enumerate(layers):
            comp.wait_event(ag_done[k])
            body(layer)
            e = torch.cuda.Event()
            e.record(comp)
            use_done[k] = e
            if k + 2 < len(layers):
                gather(k + 2)

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

    def _on_offload(self, ev: Event) -> None:
        """OffloadAct: interior checkpoints of (stage, microbatch) -> pinned host."""
        if not self.offload or self.n_tok == 0:
            return
        s, m = ev.key[1], ev.key[2]
        n = self.n_tok
        for layer in self.interior.get(s, ()):
            self.host_act[(layer, m)][:n].copy_(self.act[(layer, m)][:n], non_blocking=True)

    def _on_load(self, ev: Event) -> None:
        """LoadAct: pinned host -> the microbatch's device ring slot, before the backward."""
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
    "OptimStep": StageExecutor._noop,
    "Fwd": StageExecutor._on_fwd,
    "Recompute": StageExecutor._noop,
    "Bwd": StageExecutor._on_bwd,
    "P2PSend": StageExecutor._on_send,
    "P2PRecv": StageExecutor._noop,
    "OffloadAct": StageExecutor._on_offload,
    "LoadAct": StageExecutor._on_load,
    "FreeParams": StageExecutor._noop,
}
