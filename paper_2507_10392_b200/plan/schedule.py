"""Microbatch schedule: the plan's per-iteration task graph and its list order.

Restates the task graph of hetplan ``simulate._Builder.build``
(simulate.py:256-558) and the deterministic list scheduler of ``simulate_plan``
(simulate.py:590-649).  The reference uses them to *model* an iteration; here
they define what the B200 executor *runs*: every rank walks the global event
order filtered to the events it participates in, which is a valid static
instruction stream (each pick is the global minimum start, so per-device event
order respects every dependency).  Task keys, creation order, priorities and
durations follow the reference exactly so the event sequence is bit-identical
(pinned by tests/golden/schedule_*.json).

Memory-accounting effects of the simulator (simulate.py:660-696) are not part
of the execution contract and are not restated.
"""

from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from .configure import TrainingPlan
from .costs import CostContext, Strategy, allgather_time, best_cross_link, reduce_scatter_time

CATEGORIES = ("params", "grads", "optim", "activations")   # simulate.py:60

# Tie-break rank of each event kind (simulate.py:47-59).
KIND_RANK = {
    "AllGather": 0, "P2PRecv": 1, "LoadAct": 2, "Fwd": 3, "Recompute": 4, "Bwd": 5,
    "P2PSend": 6, "OffloadAct": 7, "FreeParams": 8, "ReduceScatter": 9, "OptimStep": 10,
}
_FORWARD_KEYS = {"F", "OA"}


class SimulationError(RuntimeError):
    """Malformed plan or a wedged task graph."""


@dataclass
class Task:
    seq: int
    key: tuple
    kind: str
    group: int
    stage: int
    microbatch: int
    layer: int
    duration: float
    lanes: Tuple[Tuple[str, str], ...]
    deps: Tuple[tuple, ...]
    prio: tuple
    effects: Tuple[Tuple[str, str, float, str], ...] = ()   # (device, category, delta, at)


@dataclass(frozen=True)
class Event:
    """One scheduled task (fields of the reference's ScheduledEvent + its key)."""

    key: tuple
    kind: str
    group: int
    stage: int
    microbatch: int
    layer: int
    start: float
    end: float
    device_ids: Tuple[str, ...]
    lane: str
    deps: Tuple[tuple, ...] = ()
    effects: Tuple[Tuple[str, str, float, str], ...] = ()


class TaskGraph:
    """Builds the task list for one iteration of ``plan``."""

    def __init__(self, ctx: CostContext, plan: TrainingPlan) -> None:
        self.ctx, self.plan = ctx, plan
        self.order = plan.global_order()
        self.ranges = plan.stage_layer_ranges()
        self.n = len(self.order)
        covered = sum(g.layers_assigned for g in plan.groups)
        if covered != ctx.model.num_layers:
            raise SimulationError(f"plan covers {covered} layers, model has {ctx.model.num_layers}")
        self.tasks: List[Task] = []
        self.by_key: Dict[tuple, Task] = {}
        self._fwd_stages = {gi: [s for s in range(self.n) if self.order[s][0] == gi]
                            for gi in range(len(plan.groups))}

    # ------------------------------------------------------------ geometry
    def group_of(self, s: int) -> int:
        return self.order[s][0]

    def layers(self, s: int) -> List[int]:
        lo, hi = self.ranges[s]
        return list(range(lo, hi))

    def ids(self, gi: int) -> Tuple[str, ...]:
        return self.plan.groups[gi].device_ids

    def lanes(self, gi: int, lane: str):
        return tuple((d, lane) for d in self.ids(gi))

    def compute_time(self, s: int, part: str) -> float:
        """Slowest member's per-microbatch time through the ministage."""
        group = self.plan.groups[self.group_of(s)]
        worst = 0.0
        for dev in group.devices:
            share = group.shares[dev.id]
            if share <= 0:
                continue
            t = 0.0
            for layer in self.layers(s):
                f = self.ctx.runtime.fit_for(dev.kind, self.ctx.model.class_of(layer))
                t += (f.fwd_alpha + f.fwd_beta * share) if part == "fwd" else \
                     (f.bwd_alpha + f.bwd_beta * share)
            worst = max(worst, t)
        return worst

    def act_unit(self, gi: int, dev_id: str) -> int:
        ctx = self.ctx
        return (self.plan.groups[gi].shares[dev_id] * ctx.workload.seq_len
                * ctx.model.hidden_size * ctx.model.bytes_per_element)

    def act_transfer_time(self, gi: int) -> float:
        return max(self.act_unit(gi, d) for d in self.ids(gi)) / self.ctx.host_transfer_bw

    def layer_bytes(self, layer: int) -> int:
        return self.ctx.model.params_of(layer) * self.ctx.model.bytes_per_element

    def ag_time(self, s: int, layer: int) -> float:
        gi = self.group_of(s)
        return allgather_time(self.ctx, self.layer_bytes(layer) / len(self.ids(gi)), self.ids(gi))

    def rs_time(self, s: int, layer: int) -> float:
        gi = self.group_of(s)
        return reduce_scatter_time(self.ctx, self.layer_bytes(layer), self.ids(gi))

    def chunk_bytes(self, s: int):
        return sum(self.layer_bytes(layer) for layer in self.layers(s))

    def z3_window_bytes(self, s: int) -> float:
        """Materialised-parameter window: the chunk's two largest layers minus the
        resident shard slice (simulate.py:223-229)."""
        d_dp = len(self.ids(self.group_of(s)))
        sizes = sorted((self.layer_bytes(layer) for layer in self.layers(s)), reverse=True)
        return sum(sizes[:2]) * (1.0 - 1.0 / d_dp)

    # ------------------------------------------------------------ emission
    def add(self, key, kind, stage, microbatch=-1, layer=-1, *, duration, lanes, deps,
            effects=()) -> None:
        if key in self.by_key:
            raise SimulationError(f"duplicate task key {key}")
        forward = key[0].endswith("f") or key[0] in _FORWARD_KEYS
        if kind == "OptimStep" or stage < 0:
            pos = 2 * self.n
        else:
            pos = stage if forward else 2 * self.n - 1 - stage
        t = Task(seq=len(self.tasks), key=key, kind=kind,
                 group=self.group_of(stage) if stage >= 0 else -1, stage=stage,
                 microbatch=microbatch, layer=layer, duration=duration, lanes=tuple(lanes),
                 deps=tuple(deps), prio=(pos, microbatch, KIND_RANK[kind], layer, len(self.tasks)),
                 effects=tuple(effects))
        self.by_key[key] = t
        self.tasks.append(t)

    def build(self) -> List[Task]:
        plan, ctx = self.plan, self.ctx
        M = plan.n_microbatches
        offload = plan.strategy.offloads
        per_mb = plan.strategy.gathers_per_microbatch
        k_act = ctx.k_act
        link: Dict[Tuple[int, str], Tuple[str, str, float]] = {}
        for b in range(self.n - 1):
            lo, hi = self.group_of(b), self.group_of(b + 1)
            if lo != hi:
                link[(b, "f")] = best_cross_link(ctx, self.ids(lo), self.ids(hi))
                link[(b, "b")] = best_cross_link(ctx, self.ids(hi), self.ids(lo))
        boundary_bytes = (plan.microbatch_size * ctx.workload.seq_len * ctx.model.hidden_size
                          * ctx.model.bytes_per_element)
        fwd_slots = {gi: [(s, m) for s in st for m in range(M)] for gi, st in self._fwd_stages.items()}
        bwd_slots = {gi: [(s, m) for s in reversed(st) for m in range(M)]
                     for gi, st in self._fwd_stages.items()}

        # ---------------- forward: gathers, Fwd, offload, boundary sends ----
        for s in range(self.n):
            gi = self.group_of(s)
            mine = self._fwd_stages[gi]
            q = mine.index(s)
            lays = self.layers(s)
            coll = self.lanes(gi, "collective")
            if per_mb:
                for m in range(M):
                    for i, layer in enumerate(lays):
                        if i > 0:
                            deps = [("AGf", s, i - 1, m)]
                        elif m > 0:
                            deps = [("F", s, m - 1)]
                        elif q >= 1:
                            deps = [("F", mine[q - 1], M - 1)]
                        else:
                            deps = []
                        eff = [(d, "params", self.z3_window_bytes(s), "start")
                               for d in self.ids(gi)] if i == 0 else []
                        self.add(("AGf", s, i, m), "AllGather", s, m, layer,
                                 duration=self.ag_time(s, layer), lanes=coll, deps=deps,
                                 effects=eff)
            else:
                for i, layer in enumerate(lays):
                    deps = [("AGf", s, i - 1)] if i > 0 else []
                    if offload and q >= 2:
                        deps.append(("FREEf", mine[q - 2]))
                    eff = [(d, "params", self.layer_bytes(layer), "start")
                           for d in self.ids(gi)] if offload else []
                    self.add(("AGf", s, i), "AllGather", s, -1, layer,
                             duration=self.ag_time(s, layer), lanes=coll, deps=deps, effects=eff)
            fwd_t = self.compute_time(s, "fwd")
            for m in range(M):
                deps = ([("AGf", s, i, m) for i in range(len(lays))] if per_mb
                        else [("AGf", s, i) for i in range(len(lays))])
                if m > 0:
                    deps.append(("F", s, m - 1))
                if s > 0:
                    deps.append(("F", s - 1, m) if self.group_of(s - 1) == gi else ("PRf", s - 1, m))
                if offload:
                    p = fwd_slots[gi].index((s, m))
                    if p >= 2:
                        deps.append(("OA",) + fwd_slots[gi][p - 2])
                eff = []
                for d in self.ids(gi):
                    # the materialised window closes on every member, zero-share included
                    if per_mb:
                        eff.append((d, "params", -self.z3_window_bytes(s), "end"))
                    u = self.act_unit(gi, d)
                    if u == 0:
                        continue
                    if offload:
                        eff.append((d, "activations", (1 + k_act) * u, "start"))
                    else:
                        eff.append((d, "activations", (len(lays) + k_act) * u, "start"))
                    eff.append((d, "activations", -k_act * u, "end"))
                self.add(("F", s, m), "Fwd", s, m, duration=fwd_t,
                         lanes=self.lanes(gi, "compute"), deps=deps, effects=eff)
                if offload:
                    self.add(("OA", s, m), "OffloadAct", s, m, duration=self.act_transfer_time(gi),
                             lanes=self.lanes(gi, "host"), deps=[("F", s, m)],
                             effects=[(d, "activations", -self.act_unit(gi, d), "end")
                                      for d in self.ids(gi) if self.act_unit(gi, d) > 0])
                if s + 1 < self.n and self.group_of(s + 1) != gi:
                    src, dst, bw = link[(s, "f")]
                    self.add(("PSf", s, m), "P2PSend", s, m, duration=boundary_bytes / bw,
                             lanes=((src, "p2p"),), deps=[("F", s, m)])
                    self.add(("PRf", s, m), "P2PRecv", s + 1, m, duration=ctx.comm.p2p_latency,
                             lanes=((dst, "p2p"),), deps=[("PSf", s, m)])
            if offload:
                self.add(("FREEf", s), "FreeParams", s, duration=0.0, lanes=(),
                         deps=[("F", s, M - 1)],
                         effects=[(d, "params", -self.chunk_bytes(s), "end") for d in self.ids(gi)])

        # ---------------- backward: gathers, reload, recompute, Bwd, RS -----
        for s in reversed(range(self.n)):
            gi = self.group_of(s)
            chunks = list(reversed(self._fwd_stages[gi]))
            r = chunks.index(s)
            lays = self.layers(s)
            coll = self.lanes(gi, "collective")
            if per_mb:
                for m in range(M):
                    for i, layer in enumerate(lays):
                        if i > 0:
                            deps = [("AGb", s, i - 1, m)]
                        else:
                            deps = [("F", s, M - 1)]
                            if m > 0:
                                deps.append(("B", s, m - 1))
                            elif r >= 1:
                                deps.append(("B", chunks[r - 1], M - 1))
                        eff = [(d, "params", self.z3_window_bytes(s), "start")
                               for d in self.ids(gi)] if i == 0 else []
                        self.add(("AGb", s, i, m), "AllGather", s, m, layer,
                                 duration=self.ag_time(s, layer), lanes=coll, deps=deps,
                                 effects=eff)
            else:
                for i, layer in enumerate(lays):
                    if i > 0:
                        deps = [("AGb", s, i - 1)]
                    elif offload:
                        deps = [("FREEf", s)]
                        if r >= 2:
                            deps.append(("FREEb", chunks[r - 2]))
                    else:
                        deps = [("F", s, M - 1)]
                    eff = [(d, "params", self.layer_bytes(layer), "start")
                           for d in self.ids(gi)] if offload else []
                    self.add(("AGb", s, i), "AllGather", s, -1, layer,
                             duration=self.ag_time(s, layer), lanes=coll, deps=deps, effects=eff)
            rc_t = self.compute_time(s, "fwd")
            bwd_t = self.compute_time(s, "bwd")
            grad_bytes = self.chunk_bytes(s) / (len(self.ids(gi)) if per_mb else 1)
            for m in range(M):
                if offload:
                    p = bwd_slots[gi].index((s, m))
                    deps = [("OA", s, m), ("RC",) + bwd_slots[gi][p - 1] if p >= 1 else ("F", s, M - 1)]
                    self.add(("LA", s, m), "LoadAct", s, m, duration=self.act_transfer_time(gi),
                             lanes=self.lanes(gi, "host"), deps=deps,
                             effects=[(d, "activations", self.act_unit(gi, d), "end")
                                      for d in self.ids(gi) if self.act_unit(gi, d) > 0])
                deps = [("F", s, m)]
                if m > 0:
                    deps.append(("B", s, m - 1))
                if offload:
                    deps.append(("LA", s, m))
                deps += ([("AGb", s, i, m) for i in range(len(lays))] if per_mb
                         else [("AGb", s, i) for i in range(len(lays))])
                if m == 0 and r >= 1:
                    prev = chunks[r - 1]
                    deps.append(("RS", prev, len(self.layers(prev)) - 1))
                self.add(("RC", s, m), "Recompute", s, m, duration=rc_t,
                         lanes=self.lanes(gi, "compute"), deps=deps,
                         effects=[(d, "activations", k_act * self.act_unit(gi, d), "start")
                                  for d in self.ids(gi) if self.act_unit(gi, d) > 0])
                deps = [("RC", s, m)]
                if s + 1 < self.n:
                    deps.append(("B", s + 1, m) if self.group_of(s + 1) == gi else ("PRb", s, m))
                eff = [(d, "grads", grad_bytes, "start") for d in self.ids(gi)] if m == 0 else []
                drop = 1 + k_act if offload else len(lays) + k_act
                eff += [(d, "activations", -drop * self.act_unit(gi, d), "end")
                        for d in self.ids(gi) if self.act_unit(gi, d) > 0]
                if per_mb:
                    eff += [(d, "params", -self.z3_window_bytes(s), "end") for d in self.ids(gi)]
                self.add(("B", s, m), "Bwd", s, m, duration=bwd_t,
                         lanes=self.lanes(gi, "compute"), deps=deps, effects=eff)
                if s > 0 and self.group_of(s - 1) != gi:
                    src, dst, bw = link[(s - 1, "b")]
                    self.add(("PSb", s - 1, m), "P2PSend", s, m, duration=boundary_bytes / bw,
                             lanes=((src, "p2p"),), deps=[("B", s, m)])
                    self.add(("PRb", s - 1, m), "P2PRecv", s - 1, m, duration=ctx.comm.p2p_latency,
                             lanes=((dst, "p2p"),), deps=[("PSb", s - 1, m)])
            if offload:
                self.add(("FREEb", s), "FreeParams", s, duration=0.0, lanes=(),
                         deps=[("B", s, M - 1)],
                         effects=[(d, "params", -self.chunk_bytes(s), "end") for d in self.ids(gi)])
            for i, layer in enumerate(lays):
                deps = [("B", s, M - 1)] + ([("RS", s, i - 1)] if i > 0 else [])
                eff = [(d, "grads", -grad_bytes, "end") for d in self.ids(gi)] \
                    if i == len(lays) - 1 else []
                self.add(("RS", s, i), "ReduceScatter", s, -1, layer,
                         duration=self.rs_time(s, layer), lanes=coll, deps=deps, effects=eff)

        # ---------------- per-ministage optimizer -------------------------
        for s in range(self.n):
            gi = self.group_of(s)
            deps = [("RS", s, i) for i in range(len(self.layers(s)))]
            if not plan.strategy.offloads:
                for other in self._fwd_stages[gi]:
                    deps += [("RS", other, i) for i in range(len(self.layers(other)))]
                deps = sorted(set(deps))
            local = sum(ctx.model.params_of(layer) for layer in self.layers(s)) / plan.groups[gi].d_dp
            self.add(("OPT", s), "OptimStep", s, duration=local * ctx.optim_update_per_param,
                     lanes=self.lanes(gi, "compute"), deps=deps)

        for t in self.tasks:
            for dep in t.deps:
                if dep not in self.by_key:
                    raise SimulationError(f"task {t.key} depends on unknown {dep}")
        return self.tasks


class OneFOneBGraph(TaskGraph):
    """1F1B microbatch schedule (BASELINE config 4) over the same plan types.

    The reference has no 1F1B (SPEC.md:477 lists it as a non-goal), so this
    schedule has no reference oracle.  It keeps the reference's task kinds,
    keys and cost model, and uses PP_ZERO3 collective semantics — one
    AllGather per layer per microbatch per pass — because 1F1B interleaves the
    forward and backward of different microbatches (SURVEY §7 hard part 7);
    the per-group AG/RS counts therefore still equal count_collectives
    (costs.py:189-201).  Each group owns exactly one ministage (one pipeline
    stage); its compute lane runs min(k-s-1, M) warm-up forwards, then
    alternates one forward / one (recompute + backward), then drains.
    """

    def build(self) -> List[Task]:
        plan, ctx = self.plan, self.ctx
        if not plan.strategy.gathers_per_microbatch:
            raise SimulationError("1F1B needs per-microbatch gathers (strategy pp-zero3)")
        if any(len(g.ministage_sizes) != 1 for g in plan.groups):
            raise SimulationError("1F1B here supports one ministage per group")
        M, k = plan.n_microbatches, self.n
        link: Dict[Tuple[int, str], Tuple[str, str, float]] = {}
        for b in range(k - 1):
            lo, hi = self.group_of(b), self.group_of(b + 1)
            link[(b, "f")] = best_cross_link(ctx, self.ids(lo), self.ids(hi))
            link[(b, "b")] = best_cross_link(ctx, self.ids(hi), self.ids(lo))
        boundary_bytes = (plan.microbatch_size * ctx.workload.seq_len * ctx.model.hidden_size
                          * ctx.model.bytes_per_element)
        for s in range(k):
            gi = self.group_of(s)
            lays = self.layers(s)
            coll = self.lanes(gi, "collective")
            comp = self.lanes(gi, "compute")
            warm = min(k - s - 1, M)
            seq = [("F", m) for m in range(warm)]
            nf, nb = warm, 0
            while nb < M:
                if nf < M:
                    seq.append(("F", nf))
                    nf += 1
                seq.append(("B", nb))
                nb += 1
            fwd_t, rc_t, bwd_t = (self.compute_time(s, "fwd"), self.compute_time(s, "fwd"),
                                  self.compute_time(s, "bwd"))
            prev = None  # previous compute task on this stage's lane
            for op, m in seq:
                tag = "AGf" if op == "F" else "AGb"
                for i, layer in enumerate(lays):
                    deps = [(tag, s, i - 1, m)] if i > 0 else ([prev] if prev else [])
                    self.add((tag, s, i, m), "AllGather", s, m, layer,
                             duration=self.ag_time(s, layer), lanes=coll, deps=deps)
                gathers = [(tag, s, i, m) for i in range(len(lays))]
                if op == "F":
                    deps = gathers + ([prev] if prev else [])
                    if s > 0:
                        deps.append(("PRf", s - 1, m))
                    self.add(("F", s, m), "Fwd", s, m, duration=fwd_t, lanes=comp, deps=deps)
                    prev = ("F", s, m)
                    if s + 1 < k:
                        src, dst, bw = link[(s, "f")]
                        self.add(("PSf", s, m), "P2PSend", s, m, duration=boundary_bytes / bw,
                                 lanes=((src, "p2p"),), deps=[("F", s, m)])
                        self.add(("PRf", s, m), "P2PRecv", s + 1, m,
                                 duration=ctx.comm.p2p_latency, lanes=((dst, "p2p"),),
                                 deps=[("PSf", s, m)])
                else:
                    deps = gathers + [("F", s, m)] + ([prev] if prev else [])
                    self.add(("RC", s, m), "Recompute", s, m, duration=rc_t, lanes=comp, deps=deps)
                    deps = [("RC", s, m)] + ([("PRb", s, m)] if s + 1 < k else [])
                    self.add(("B", s, m), "Bwd", s, m, duration=bwd_t, lanes=comp, deps=deps)
                    prev = ("B", s, m)
                    if s > 0:
                        src, dst, bw = link[(s - 1, "b")]
                        self.add(("PSb", s - 1, m), "P2PSend", s, m, duration=boundary_bytes / bw,
                                 lanes=((src, "p2p"),), deps=[("B", s, m)])
                        self.add(("PRb", s - 1, m), "P2PRecv", s - 1, m,
                                 duration=ctx.comm.p2p_latency, lanes=((dst, "p2p"),),
                                 deps=[("PSb", s - 1, m)])
            for i, layer in enumerate(lays):
                deps = [prev] + ([("RS", s, i - 1)] if i > 0 else [])
                self.add(("RS", s, i), "ReduceScatter", s, -1, layer,
                         duration=self.rs_time(s, layer), lanes=coll, deps=deps)
            local = sum(ctx.model.params_of(layer) for layer in lays) / plan.groups[gi].d_dp
            self.add(("OPT", s), "OptimStep", s, duration=local * ctx.optim_update_per_param,
                     lanes=comp, deps=[("RS", s, i) for i in range(len(lays))])
        for t in self.tasks:
            for dep in t.deps:
                if dep not in self.by_key:
                    raise SimulationError(f"task {t.key} depends on unknown {dep}")
        return self.tasks


def list_schedule(tasks: Sequence[Task], plan: TrainingPlan) -> List[Event]:
    """Greedy list scheduling: repeatedly start the ready task with the least
    (earliest start, priority); a task occupies all its lanes."""
    waiting = {t.key: len(t.deps) for t in tasks}
    children: Dict[tuple, List[Task]] = defaultdict(list)
    for t in tasks:
        for dep in t.deps:
            children[dep].append(t)
    lane_free: Dict[Tuple[str, str], float] = defaultdict(float)
    earliest = {t.key: 0.0 for t in tasks}
    ready = [t for t in tasks if not t.deps]
    out: List[Event] = []
    while ready:
        def start_of(t: Task) -> float:
            s = earliest[t.key]
            for ln in t.lanes:
                if lane_free[ln] > s:
                    s = lane_free[ln]
            return s

        pick = min(ready, key=lambda t: (start_of(t), t.prio))
        start = start_of(pick)
        end = start + pick.duration
        for ln in pick.lanes:
            lane_free[ln] = end
        ready.remove(pick)
        out.append(Event(key=pick.key, kind=pick.kind, group=pick.group, stage=pick.stage,
                         microbatch=pick.microbatch, layer=pick.layer, start=start, end=end,
                         device_ids=tuple(d for d, _ in pick.lanes) or plan.groups[pick.group].device_ids,
                         lane=pick.lanes[0][1] if pick.lanes else "none", deps=pick.deps,
                         effects=pick.effects))
        for child in children[pick.key]:
            waiting[child.key] -= 1
            if end > earliest[child.key]:
                earliest[child.key] = end
            if waiting[child.key] == 0:
                ready.append(child)
    if len(out) != len(tasks):
        done = {e.key for e in out}
        stuck = [t.key for t in tasks if t.key not in done][:8]
        raise SimulationError(f"simulation deadlocked with {len(tasks) - len(out)} tasks blocked; "
                              f"first stuck: {stuck}")
    return out


@dataclass
class Schedule:
    """The iteration's global event order plus derived per-device streams."""

    plan: TrainingPlan
    events: List[Event]

    @property
    def iteration_time(self) -> float:
        return max(e.end for e in self.events)

    def collective_counts(self) -> Dict[int, Dict[str, int]]:
        counts = {gi: {"allgather": 0, "reduce_scatter": 0} for gi in range(len(self.plan.groups))}
        for e in self.events:
            if e.kind == "AllGather":
                counts[e.group]["allgather"] += 1
            elif e.kind == "ReduceScatter":
                counts[e.group]["reduce_scatter"] += 1
        return counts

    def memory(self, ctx: CostContext):
        """(peaks, traces) of the simulator's memory accounting for this schedule."""
        return memory_replay(ctx, self.plan, self.events)

    def gantt_rows(self):
        return [(e.start, e.end, e.kind, e.group, e.stage, e.microbatch, e.layer, e.lane,
                 e.device_ids) for e in self.events]

    def group_of_device(self, dev_id: str) -> int:
        for gi, g in enumerate(self.plan.groups):
            if dev_id in g.device_ids:
                return gi
        raise KeyError(dev_id)

    def stream_for(self, dev_id: str) -> List[Event]:
        """Events device ``dev_id`` executes, in global order.

        Every task is tagged with the group of its stage (simulate.py:236).  On
        B200 a boundary transfer is many-to-many — every member of the sending
        group holds part of the microbatch and every member of the receiving
        group needs part of it — and it is ONE global operation: the receiving
        group posts its receives at the P2PSend event (its P2PRecv event only
        marks arrival).  With every NCCL operation (group collective or
        transfer) at a single position of one global order, the earliest
        unfinished operation always has all its participants' earlier work
        done, so blocking sends can never form a cycle.
        """
        gi = self.group_of_device(dev_id)
        order = self.plan.global_order()
        out = []
        for e in self.events:
            if e.group == gi:
                out.append(e)
            elif e.kind == "P2PSend":
                b = e.key[1]  # boundary between global stages b and b+1
                peer_stage = b + 1 if e.key[0] == "PSf" else b
                if order[peer_stage][0] == gi:
                    out.append(e)  # receiving side of the transfer
        return out


def initial_memory(ctx: CostContext, plan: TrainingPlan) -> Dict[str, Dict[str, float]]:
    """Resident-from-t=0 bytes per device and category (simulate.py:565-588):
    optimizer shard, persistent gradient buffer, strategy-dependent parameters."""
    base: Dict[str, Dict[str, float]] = {}
    elem = ctx.model.bytes_per_element
    ranges = plan.stage_layer_ranges()
    order = plan.global_order()
    for gi, group in enumerate(plan.groups):
        layers = [layer for idx, (g, _) in enumerate(order) if g == gi
                  for layer in range(*ranges[idx])]
        param_count = sum(ctx.model.params_of(layer) for layer in layers)
        param_bytes = param_count * elem
        d_dp = group.d_dp
        for dev in group.devices:
            state = {c: 0.0 for c in CATEGORIES}
            state["optim"] = param_count * ctx.workload.optimizer_bytes_per_param / d_dp
            state["grads"] = param_bytes / d_dp
            if plan.strategy is Strategy.PP_ZERO2:
                state["params"] = param_bytes
            elif plan.strategy is Strategy.PP_ZERO3:
                state["params"] = param_bytes / d_dp
            base[dev.id] = state
    return base


def memory_replay(ctx: CostContext, plan: TrainingPlan, events: Sequence[Event]):
    """The simulator's memory accounting (simulate.py:660-696): apply every event's
    effects in time order — end-effects before start-effects at equal timestamps —
    on top of the initial residency.  Returns (peaks {device: {category|total}},
    traces {device: [(time, params, grads, optim, activations, total)]})."""
    deltas: Dict[str, List[tuple]] = defaultdict(list)
    for idx, e in enumerate(events):
        for dev, cat, delta, at in e.effects:
            time = e.start if at == "start" else e.end
            phase = 1 if at == "start" else 0
            deltas[dev].append((time, phase, idx, cat, delta))
    base = initial_memory(ctx, plan)
    peaks: Dict[str, Dict[str, float]] = {}
    traces: Dict[str, List[tuple]] = {}
    for group in plan.groups:
        for dev in group.devices:
            state = dict(base[dev.id])
            trace = [(0.0, state["params"], state["grads"], state["optim"],
                      state["activations"], sum(state.values()))]
            peak = dict(state)
            peak["total"] = sum(state.values())
            for time, _, _, cat, delta in sorted(deltas.get(dev.id, [])):
                state[cat] += delta
                total = sum(state.values())
                trace.append((time, state["params"], state["grads"], state["optim"],
                              state["activations"], total))
                for c in CATEGORIES:
                    peak[c] = max(peak[c], state[c])
                peak["total"] = max(peak["total"], total)
            for cat, value in state.items():
                if value < -1e-6 or (cat in ("params", "activations")
                                     and abs(value - base[dev.id][cat]) > 1e-6):
                    raise SimulationError(f"memory accounting leak on {dev.id}/{cat}: "
                                          f"end state {value}, expected {base[dev.id][cat]}")
            peaks[dev.id] = peak
            traces[dev.id] = trace
    return peaks, traces


def write_gantt_csv(path: str, rows) -> None:
    """Gantt CSV in the reference's columns (simulate.py:115-126); rows are
    (start, end, kind, group, stage, microbatch, layer, lane, devices)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["start", "end", "kind", "group", "stage", "microbatch", "layer", "lane",
                    "devices"])
        for r in rows:
            w.writerow([repr(r[0]), repr(r[1])] + list(r[2:8]) + [" ".join(r[8])])


def write_memory_csv(path: str, traces) -> None:
    """Memory CSV in the reference's columns (simulate.py:128-137)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["device", "time", "params", "grads", "optim", "activations", "total"])
        for dev in sorted(traces):
            for row in traces[dev]:
                w.writerow([dev] + [repr(v) for v in row])


def build_schedule(ctx: CostContext, plan: TrainingPlan, kind: str = "gpipe") -> Schedule:
    """kind "gpipe": the reference's ministage-interleaved GPipe schedule
    (simulate.py:256-558, bit-exact); "1f1b": OneFOneBGraph."""
    graph = {"gpipe": TaskGraph, "1f1b": OneFOneBGraph}[kind](ctx, plan)
    return Schedule(plan=plan, events=list_schedule(graph.build(), plan))
