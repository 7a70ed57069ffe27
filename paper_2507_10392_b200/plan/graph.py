"""Cluster bandwidth graph and device partitions (planner Phase 1 inputs).

Restates the data types of hetplan ``partition.py`` the plan layer needs:
``ClusterGraph`` (partition.py:47-101), ``Partition`` (:104-126),
``make_partition`` (:133-140) and ``build_cluster_graph`` (:137-145).  The
min-k-cut search itself lives in ``mincut.py``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import FrozenSet, Iterable, Sequence, Tuple

import numpy as np

from .workload import ClusterProfile


class PartitionError(ValueError):
    """Invalid partitioning request."""


class ClusterGraph:
    """Complete graph over devices, edge weight = link bandwidth (bytes/s)."""

    def __init__(self, vertices: Sequence[str], weights) -> None:
        self.vertices = tuple(vertices)
        n = len(self.vertices)
        self.weights = np.asarray(weights, dtype=np.float64)
        if self.weights.shape != (n, n):
            raise PartitionError("weight matrix shape does not match vertex count")
        if len(set(self.vertices)) != n:
            raise PartitionError("duplicate vertex ids")
        self._index = {v: i for i, v in enumerate(self.vertices)}
        # rank of each slot in lexicographic id order (min-cut tie-breaks)
        self._lexrank = np.empty(n, dtype=np.int64)
        for rank, slot in enumerate(sorted(range(n), key=lambda i: self.vertices[i])):
            self._lexrank[slot] = rank
        self._minbw_cache: dict = {}
        self._crosslink_cache: dict = {}

    def __len__(self) -> int:
        return len(self.vertices)

    def index_of(self, vertex: str) -> int:
        return self._index[vertex]

    def edge_weight(self, u: str, v: str) -> float:
        return float(self.weights[self._index[u], self._index[v]])

    def crossing_weight(self, groups: Sequence[Iterable[str]]) -> float:
        """Sum of edges between different groups, accumulated over i<j slots."""
        label = np.empty(len(self.vertices), dtype=np.int64)
        for gi, g in enumerate(groups):
            for v in g:
                label[self._index[v]] = gi
        total = 0.0
        n = len(self.vertices)
        for i in range(n):
            for j in range(i + 1, n):
                if label[i] != label[j]:
                    total += float(self.weights[i, j])
        return total


@dataclass(frozen=True)
class Partition:
    k: int
    groups: Tuple[FrozenSet[str], ...]
    cut_weight: float

    def __post_init__(self) -> None:
        if self.k != len(self.groups):
            raise PartitionError("k does not match number of groups")
        if any(len(g) == 0 for g in self.groups):
            raise PartitionError("empty group in partition")
        members = [v for g in self.groups for v in g]
        if len(members) != len(set(members)):
            raise PartitionError("groups are not disjoint")

    def group_of(self, vertex: str) -> int:
        for gi, g in enumerate(self.groups):
            if vertex in g:
                return gi
        raise KeyError(vertex)


def make_partition(graph: ClusterGraph, groups: Sequence[Iterable[str]]) -> Partition:
    ordered = tuple(sorted((frozenset(g) for g in groups), key=min))
    if {v for g in ordered for v in g} != set(graph.vertices):
        raise PartitionError("groups do not cover the vertex set exactly")
    return Partition(k=len(ordered), groups=ordered, cut_weight=graph.crossing_weight(ordered))


def build_cluster_graph(profile: ClusterProfile) -> ClusterGraph:
    devs = profile.devices
    n = len(devs)
    w = np.zeros((n, n), dtype=np.float64)
    for i in range(n):
        for j in range(i + 1, n):
            w[i, j] = w[j, i] = profile.bandwidth(devs[i], devs[j])
    return ClusterGraph([d.id for d in devs], w)
