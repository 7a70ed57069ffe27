"""Strategy, cost context and the collective / P2P cost formulas.

Restates hetplan ``costs.py``: ``Strategy`` (costs.py:42-60), ``CommParams`` /
``CostContext`` (:63-82), the estimate records (:85-118), ring AllGather /
ReduceScatter times (:138-158), the best cross link (:161-178), P2P time
(:181-186) and the exact collective-count invariant (:189-201).  The schedule
derives task durations — and therefore the executor's instruction order —
from these, so the arithmetic follows the reference operation for operation.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum
from typing import Sequence, Tuple

import numpy as np

from .graph import ClusterGraph
from .workload import LayerRuntimeModel, ModelSpec, WorkloadSpec


class Strategy(Enum):
    INTERLEAVED = "zorse"   # ministage-interleaved PP, gather once per layer per pass
    PP_ZERO2 = "pp-zero2"
    PP_ZERO3 = "pp-zero3"   # re-gather per layer per microbatch

    @property
    def offloads(self) -> bool:
        return self is Strategy.INTERLEAVED

    @property
    def gathers_per_microbatch(self) -> bool:
        return self is Strategy.PP_ZERO3


@dataclass(frozen=True)
class CommParams:
    ring_latency_per_hop: float = 50e-6
    p2p_latency: float = 100e-6


@dataclass(frozen=True)
class CostContext:
    graph: ClusterGraph
    runtime: LayerRuntimeModel
    model: ModelSpec
    workload: WorkloadSpec
    comm: CommParams = CommParams()
    k_act: float = 2.0
    optim_update_per_param: float = 1e-10
    host_transfer_bw: float = 12e9


@dataclass(frozen=True)
class LatencyEstimate:
    l_forwards: float
    l_backwards: float
    l_startup: float
    n_ministages: int
    l_total: float = field(init=False)

    def __post_init__(self) -> None:
        object.__setattr__(self, "l_total",
                           (self.l_forwards + self.l_backwards) * self.n_ministages + self.l_startup)


@dataclass(frozen=True)
class MemoryEstimate:
    m_params: float
    m_grads: float
    m_optim: float
    m_activations: float
    m_total: float = field(init=False)

    def __post_init__(self) -> None:
        object.__setattr__(self, "m_total",
                           self.m_params + self.m_grads + self.m_optim + self.m_activations)


def min_internal_bw(graph: ClusterGraph, device_ids: Sequence[str]) -> float:
    """Slowest link inside a device set (the ring bottleneck); memoised."""
    key = tuple(device_ids)
    if len(key) < 2:
        raise ValueError("bandwidth undefined for a single-device set")
    hit = graph._minbw_cache.get(key)
    if hit is None:
        idx = [graph.index_of(d) for d in key]
        sub = graph.weights[np.ix_(idx, idx)]
        hit = float(np.min(sub[np.triu_indices(len(idx), k=1)]))
        graph._minbw_cache[key] = hit
    return hit


def allgather_time(ctx: CostContext, bytes_per_shard: float, device_ids: Sequence[str]) -> float:
    g = len(device_ids)
    if g <= 1:
        return 0.0
    bw = min_internal_bw(ctx.graph, device_ids)
    total = g * bytes_per_shard
    return (g - 1) / g * total / bw + (g - 1) * ctx.comm.ring_latency_per_hop


def reduce_scatter_time(ctx: CostContext, bytes_total: float, device_ids: Sequence[str]) -> float:
    g = len(device_ids)
    if g <= 1:
        return 0.0
    bw = min_internal_bw(ctx.graph, device_ids)
    return (g - 1) / g * bytes_total / bw + (g - 1) * ctx.comm.ring_latency_per_hop


def best_cross_link(ctx: CostContext, src_ids: Sequence[str],
                    dst_ids: Sequence[str]) -> Tuple[str, str, float]:
    """Fastest (src, dst) pair: first strict maximum in row-major id order."""
    if not src_ids or not dst_ids:
        raise ValueError("empty device set for cross link")
    key = (tuple(src_ids), tuple(dst_ids))
    hit = ctx.graph._crosslink_cache.get(key)
    if hit is None:
        rows = [ctx.graph.index_of(u) for u in key[0]]
        cols = [ctx.graph.index_of(v) for v in key[1]]
        sub = ctx.graph.weights[np.ix_(rows, cols)]
        i, j = divmod(int(np.argmax(sub)), len(cols))
        hit = (key[0][i], key[1][j], float(sub[i, j]))
        ctx.graph._crosslink_cache[key] = hit
    return hit


def p2p_transfer_time(ctx: CostContext, bytes_payload: float, src_ids: Sequence[str],
                      dst_ids: Sequence[str]) -> float:
    return bytes_payload / best_cross_link(ctx, src_ids, dst_ids)[2] + ctx.comm.p2p_latency


def count_collectives(n_layers: int, n_microbatches: int, strategy: Strategy) -> Tuple[int, int]:
    """(AllGathers, ReduceScatters) per iteration for one group's layers."""
    passes = 2 * n_layers
    return (passes * n_microbatches if strategy.gathers_per_microbatch else passes), n_layers
