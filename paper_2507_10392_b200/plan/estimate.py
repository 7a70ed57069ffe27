"""Eq.1 latency and Eq.2 memory estimates used by the planner's candidate sweep.

Restates hetplan costs.py:204-615 — per-ministage compute / collective / P2P
quantities, the pipelined phase recurrence (chain, lane and head bounds),
``total_iteration_latency`` and ``memory_estimate`` / ``memory_fits``.  The
floating-point expressions keep the reference's operation order and int/float
types, so a plan selected here is byte-identical to the reference's plan file
(pinned by tests/golden/plans.json, kind "plan_training").
"""

from __future__ import annotations

import ctypes
from typing import TYPE_CHECKING, Dict, List, Optional, Sequence, Tuple

from .costs import (CostContext, LatencyEstimate, MemoryEstimate, Strategy, allgather_time,
                    p2p_transfer_time, reduce_scatter_time)
from .workload import GpuDevice

if TYPE_CHECKING:  # pragma: no cover
    from .configure import TrainingPlan


class _PlanView:
    """Cached geometry of one plan for the estimators."""

    def __init__(self, ctx: CostContext, plan: "TrainingPlan"):
        self.ctx, self.plan = ctx, plan
        self.order = plan.global_order()
        self.ranges = plan.stage_layer_ranges()
        self.n = len(self.order)
        self._pm_cache = {}

    def layers(self, s: int) -> range:
        return range(*self.ranges[s])

    def group(self, s: int):
        return self.plan.groups[self.order[s][0]]

    def per_microbatch(self, s: int, part: str) -> float:
        """Slowest member's time for one microbatch through ministage s.
        part: "fwd", "bwd" (fwd recompute + gradient) or "bwd_only".

        Members with the same (kind, share) produce the identical float, so each
        distinct pair is accumulated once (the max is unchanged, bit for bit);
        the per-layer terms are added in layer order exactly as the reference
        does (costs.py:220-249) — this is the planner's hot loop."""
        ctx, g = self.ctx, self.group(s)
        key = (s, part)
        hit = self._pm_cache.get(key)
        if hit is not None:
            return hit
        classes = [ctx.model.class_of(layer) for layer in self.layers(s)]
        worst = 0.0
        seen = set()
        for dev in g.devices:
            share = g.shares[dev.id]
            if share <= 0 or (dev.kind, share) in seen:
                continue
            seen.add((dev.kind, share))
            t = 0.0
            for cls in classes:
                f = ctx.runtime.fit_for(dev.kind, cls)
                fwd = f.fwd_alpha + f.fwd_beta * share
                bwd = f.bwd_alpha + f.bwd_beta * share
                t += fwd if part == "fwd" else (fwd + bwd if part == "bwd" else bwd)
            worst = max(worst, t)
        self._pm_cache[key] = worst
        return worst

    def gathers(self, s: int) -> List[float]:
        g = self.group(s)
        elem = self.ctx.model.bytes_per_element
        return [allgather_time(self.ctx, self.ctx.model.params_of(layer) * elem / len(g.devices),
                               g.device_ids) for layer in self.layers(s)]

    def scatter(self, s: int) -> float:
        g = self.group(s)
        elem = self.ctx.model.bytes_per_element
        total = 0.0
        for layer in self.layers(s):
            total += reduce_scatter_time(self.ctx, self.ctx.model.params_of(layer) * elem, g.device_ids)
        return total

    def boundary_p2p(self) -> List[float]:
        ctx, plan = self.ctx, self.plan
        act = plan.microbatch_size * ctx.workload.seq_len * ctx.model.hidden_size * \
            ctx.model.bytes_per_element
        out = [0.0]
        for i in range(1, self.n):
            a, b = self.order[i - 1][0], self.order[i][0]
            out.append(0.0 if a == b else p2p_transfer_time(ctx, act, plan.groups[a].device_ids,
                                                            plan.groups[b].device_ids))
        return out


def _stage_index(plan: "TrainingPlan", gi: int, rnd: int) -> int:
    try:
        return plan.global_order().index((gi, rnd))
    except ValueError:
        raise IndexError(f"no ministage (group={gi}, round={rnd})") from None


def stage_latency(ctx: CostContext, plan: "TrainingPlan", group_index: int, round_index: int,
                  direction: str = "fwd") -> float:
    """One ministage round (all microbatches) of one group (costs.py:289-320)."""
    v = _PlanView(ctx, plan)
    s = _stage_index(plan, group_index, round_index)
    m = plan.n_microbatches
    mb = v.per_microbatch(s, direction)
    ag = v.gathers(s)
    rs = v.scatter(s) if direction == "bwd" else 0.0
    p2p = v.boundary_p2p()
    d_in = p2p[s]
    d_out = p2p[s + 1] if s + 1 < v.n else 0.0
    if plan.strategy.gathers_per_microbatch:
        return max(m * (mb + sum(ag)) + rs, m * d_in, m * d_out)
    return max(m * mb, sum(ag), m * d_in, m * d_out) + rs


def phase_makespan(groups_seq, chain_mb, lane_round, head_round, rs_tail, d_in, floors,
                   start) -> Tuple[float, Dict[int, float]]:
    """Completion of one pipelined pass (costs.py:323-360): each stage's round
    ends no earlier than (chain) one traversal after the upstream stage's last
    microbatch, (lane) a full round after its group's previous round, (head)
    a round after its first microbatch could begin."""
    t_chain = start
    t_first = start
    lane_end: Dict[int, float] = {}
    for i, g in enumerate(groups_seq):
        begin = max(t_first + d_in[i], floors[i], lane_end.get(g, 0.0))
        end = max(t_chain + chain_mb[i] + d_in[i], begin + head_round[i])
        if g in lane_end:
            end = max(end, lane_end[g] + lane_round[i])
        lane_end[g] = end + rs_tail[i]
        t_chain = end
        t_first = begin + chain_mb[i]
    return t_chain, lane_end


def _native_eq1():
    from .mincut import native_kernel
    if native_kernel() is None:      # library absent: the Python restatement below
        return None
    from .._lib import lib
    return lib().zb_eq1_latency


def _fit_table(ctx: CostContext):
    """(kind index, class index, flat fits) of the runtime model, cached on it."""
    rt = ctx.runtime
    tab = getattr(rt, "_zb_fit_table", None)
    if tab is None:
        kinds = sorted({k for k, _ in rt.fits})
        classes = sorted({c for _, c in rt.fits})
        flat = []
        for k in kinds:
            for c in classes:
                f = rt.fits.get((k, c))
                flat += [f.fwd_alpha, f.fwd_beta, f.bwd_alpha, f.bwd_beta] if f else [0.0] * 4
        tab = ({k: i for i, k in enumerate(kinds)}, {c: i for i, c in enumerate(classes)},
               (ctypes.c_double * len(flat))(*flat), len(classes))
        rt._zb_fit_table = tab
    return tab


def total_iteration_latency(ctx: CostContext, plan: "TrainingPlan") -> LatencyEstimate:
    """Eq.1: forward pass + backward pass + trailing optimizer (costs.py:384-535).

    The per-microbatch compute times and the phase recurrences run in C++
    (csrc/eq1.cpp, ``zb_eq1_latency``) when the library is present — bit-identical
    to ``total_iteration_latency_py`` (tests/test_plan_units.py) — like the
    reference's compiled min-cut with its Python twin (partition.py:26-38)."""
    fn = _native_eq1()
    if fn is None:
        return total_iteration_latency_py(ctx, plan)
    v = _PlanView(ctx, plan)
    n = v.n
    kind_ix, cls_ix, fits, n_cls = _fit_table(ctx)
    grp, q, lay_off, lay_cls, mem_off, mem_kind, mem_share = [], [], [0], [], [0], [], []
    ag, rs, params = [], [], []
    members = {}
    for s, (g, qq) in enumerate(v.order):
        grp.append(g)
        q.append(qq)
        layers = v.layers(s)
        lay_cls += [cls_ix[ctx.model.class_of(layer)] for layer in layers]
        lay_off.append(len(lay_cls))
        mem = members.get(g)
        if mem is None:
            group, seen, mem = plan.groups[g], set(), []
            for dev in group.devices:
                share = group.shares[dev.id]
                if share <= 0 or (dev.kind, share) in seen:
                    continue
                seen.add((dev.kind, share))
                mem.append((kind_ix[dev.kind], share))
            members[g] = mem
        for k, share in mem:
            mem_kind.append(k)
            mem_share.append(share)
        mem_off.append(len(mem_kind))
        ag.append(sum(v.gathers(s)))
        rs.append(v.scatter(s))
        params.append(float(sum(ctx.model.params_of(layer) for layer in layers)))
    p2p = v.boundary_p2p()
    I = lambda xs: (ctypes.c_int * len(xs))(*xs)  # noqa: E731,E741
    D = lambda xs: (ctypes.c_double * len(xs))(*xs)  # noqa: E731
    out = (ctypes.c_double * 3)()
    sizes = [len(g.devices) for g in plan.groups]
    rc = fn(n, plan.n_microbatches, int(plan.strategy.gathers_per_microbatch),
            int(plan.strategy.offloads), plan.n_ministage_rounds, I(grp), I(q), I(lay_off),
            I(lay_cls), I(mem_off), I(mem_kind), I(mem_share), n_cls, fits, D(ag), D(rs), D(p2p),
            D(params), len(sizes), I(sizes), ctypes.c_double(ctx.optim_update_per_param), out)
    if rc:
        from .._lib import lib
        raise ValueError(lib().zb_last_error().decode())
    return LatencyEstimate(l_forwards=out[0], l_backwards=out[1], l_startup=out[2],
                           n_ministages=plan.n_ministage_rounds)


def total_iteration_latency_py(ctx: CostContext, plan: "TrainingPlan") -> LatencyEstimate:
    """Eq.1 in Python (the restatement the C++ path is pinned against)."""
    v = _PlanView(ctx, plan)
    n, m = v.n, plan.n_microbatches
    z3 = plan.strategy.gathers_per_microbatch
    grp = [g for g, _ in v.order]
    ag = [sum(v.gathers(s)) for s in range(n)]
    rs = [v.scatter(s) for s in range(n)]
    p2p = v.boundary_p2p()
    f_mb = [v.per_microbatch(s, "fwd") for s in range(n)]
    b_mb = [v.per_microbatch(s, "bwd") for s in range(n)]
    b_only = [v.per_microbatch(s, "bwd_only") for s in range(n)]

    def round_cost(s: int, per_mb: float, out_xfer: float) -> float:
        if z3:
            return max(m * (per_mb + ag[s]), m * out_xfer)
        return max(m * per_mb, ag[s], m * out_xfer)

    # forward
    floors_f = [0.0] * n
    chain_f = list(f_mb)
    if z3:
        for s, (g, q) in enumerate(v.order):
            if q > 0:
                chain_f[s] += ag[s]
    else:
        acc: Dict[int, float] = {}
        for s, (g, q) in enumerate(v.order):
            if q <= 1:
                acc[g] = acc.get(g, 0.0) + ag[s]
                floors_f[s] = acc[g]
    rounds_f = [round_cost(s, f_mb[s], p2p[s + 1] if s + 1 < n else 0.0) for s in range(n)]
    t_fwd, _ = phase_makespan(grp, chain_f, rounds_f, rounds_f, [0.0] * n, p2p, floors_f, 0.0)

    # backward (stages in reverse)
    rev = list(reversed(range(n)))
    d_in_b = [0.0 if k == 0 else p2p[s + 1] for k, s in enumerate(rev)]
    floors_b = [0.0] * n
    if not z3:
        floors_b[0] = t_fwd + ag[rev[0]]
    chain_b, heads_b, lanes_b = [], [], []
    visited = set()
    for k, s in enumerate(rev):
        g = grp[s]
        first_here = g not in visited
        visited.add(g)
        lane = round_cost(s, b_mb[s], p2p[s])
        lanes_b.append(lane)
        recompute = b_mb[s] - b_only[s]
        if k == 0:
            chain_b.append(b_mb[s] + (ag[s] if z3 else 0.0))
            heads_b.append(lane)
        elif first_here:
            chain_b.append(b_only[s])
            heads_b.append(max(lane - recompute, m * b_only[s]))
        else:
            chain_b.append(b_only[s] + (ag[s] if z3 else 0.0))
            heads_b.append(lane)
    _, lane_end = phase_makespan([grp[s] for s in rev], chain_b, lanes_b, heads_b,
                                 [rs[s] for s in rev], d_in_b, floors_b, t_fwd)

    # optimizer after each group's final round
    first_chunk: Dict[int, int] = {}
    all_chunks: Dict[int, float] = {}
    for s, (g, q) in enumerate(v.order):
        params = sum(ctx.model.params_of(layer) for layer in v.layers(s))
        if q == 0:
            first_chunk[g] = params
        all_chunks[g] = all_chunks.get(g, 0.0) + params
    t_total = 0.0
    for g, end in lane_end.items():
        local = first_chunk[g] if plan.strategy.offloads else all_chunks[g]
        t_total = max(t_total, end + local / len(plan.groups[g].devices) * ctx.optim_update_per_param)
    g0 = plan.groups[grp[0]]
    startup = ag[0] + rs[0] + first_chunk[grp[0]] / len(g0.devices) * ctx.optim_update_per_param
    rounds = plan.n_ministage_rounds
    return LatencyEstimate(l_forwards=(t_fwd - ag[0]) / rounds,
                           l_backwards=(t_total - t_fwd + ag[0] - startup) / rounds,
                           l_startup=startup, n_ministages=rounds)


def memory_estimate(ctx: CostContext, plan: "TrainingPlan", group_index: int, device_id: str,
                    strategy: Optional[Strategy] = None) -> MemoryEstimate:
    """Eq.2 per-GPU peak memory (costs.py:538-607)."""
    strategy = plan.strategy if strategy is None else strategy
    v = _PlanView(ctx, plan)
    group = plan.groups[group_index]
    d_dp = len(group.devices)
    elem = ctx.model.bytes_per_element
    mine = [s for s, (g, _) in enumerate(v.order) if g == group_index]
    chunk_bytes = [sum(ctx.model.params_of(layer) for layer in v.layers(s)) * elem for s in mine]
    layers = [layer for s in mine for layer in v.layers(s)]
    total_bytes = sum(ctx.model.params_of(layer) for layer in layers) * elem
    if strategy is Strategy.INTERLEAVED:
        m_params = chunk_bytes[0] if len(chunk_bytes) == 1 else \
            max(chunk_bytes[i] + chunk_bytes[i + 1] for i in range(len(chunk_bytes) - 1))
    elif strategy is Strategy.PP_ZERO2:
        m_params = total_bytes
    else:
        biggest = sorted((ctx.model.params_of(layer) * elem for layer in layers), reverse=True)
        held = sum(biggest[:2])
        m_params = held + (total_bytes - held) / d_dp
    active = max(chunk_bytes)
    if strategy is Strategy.PP_ZERO3:
        active /= d_dp
    m_grads = active + total_bytes / d_dp
    count = sum(ctx.model.params_of(layer) for layer in layers)
    m_optim = count * ctx.workload.optimizer_bytes_per_param / d_dp
    unit = group.shares[device_id] * ctx.workload.seq_len * ctx.model.hidden_size * elem
    if strategy.offloads:
        m_act = (2 + ctx.k_act) * unit
    else:
        m_act = (plan.n_microbatches * len(layers) + ctx.k_act) * unit
    return MemoryEstimate(m_params=m_params, m_grads=m_grads, m_optim=m_optim, m_activations=m_act)


def memory_fits(estimate: MemoryEstimate, gpu: GpuDevice, headroom: float = 0.9) -> bool:
    return estimate.m_total <= headroom * gpu.mem_capacity
