"""Phase-1 partitioning: Stoer-Wagner global min 2-cut and the SPLIT k-cut.

Restates hetplan ``_mincut_py.min_cut_kernel`` (_mincut_py.py:19-73, twin of
the Cython kernel _mincut_c.pyx:16-82) and ``split_min_k_cut_sequence``
(partition.py:148-237).  The numpy vector updates are the same elementwise
operations in the same order, so cut weights and sides are bit-identical to
the reference's (ties broken toward the smallest lexicographic vertex id).
"""

from __future__ import annotations

import ctypes
from typing import Dict, List, Tuple

import numpy as np

from .graph import ClusterGraph, Partition, PartitionError, make_partition


_UNRESOLVED = object()
_native = _UNRESOLVED


def native_kernel():
    """``zb_min_cut`` from the C-ABI library (csrc/mincut.cpp), or None when the library
    is not built — the reference likewise prefers its compiled kernel and falls back to
    the numpy twin (partition.py:26-38).  Resolved on the first min-cut, not at import,
    so importing the planner never loads the library."""
    global _native
    if _native is _UNRESOLVED:
        try:
            from .._lib import lib
            _native = lib().zb_min_cut
        except Exception:  # noqa: BLE001 - library absent: use the restatement below
            _native = None
    return _native


def min_cut_kernel(weights: np.ndarray, lexrank: np.ndarray) -> Tuple[float, List[int]]:
    """Global minimum 2-cut of a dense symmetric graph: (weight, sorted side)."""
    if native_kernel() is not None:
        return min_cut_native(weights, lexrank)
    return min_cut_python(weights, lexrank)


def min_cut_native(weights: np.ndarray, lexrank: np.ndarray) -> Tuple[float, List[int]]:
    w = np.ascontiguousarray(weights, dtype=np.float64)
    n = w.shape[0]
    if n < 2:
        raise ValueError("min cut needs >= 2 vertices")
    rank = np.ascontiguousarray(lexrank, dtype=np.int64)
    cut = ctypes.c_double()
    side = np.zeros(n, dtype=np.int64)
    ln = ctypes.c_int64()
    rc = native_kernel()(w.ctypes.data, n, rank.ctypes.data, ctypes.byref(cut), side.ctypes.data,
                 ctypes.byref(ln))
    if rc:
        from .._lib import lib
        raise ValueError(lib().zb_last_error().decode())
    return float(cut.value), [int(x) for x in side[:ln.value]]


def min_cut_python(weights: np.ndarray, lexrank: np.ndarray) -> Tuple[float, List[int]]:
    """Global minimum 2-cut of a dense symmetric graph: (weight, sorted side)."""
    w = np.array(weights, dtype=np.float64, copy=True)
    n = w.shape[0]
    if n < 2:
        raise ValueError("min cut needs >= 2 vertices")
    rank = np.array(lexrank, dtype=np.int64, copy=True)  # smallest member rank per supervertex
    alive = np.ones(n, dtype=bool)
    members: List[List[int]] = [[i] for i in range(n)]
    best_w, best_side = np.inf, []
    for remaining in range(n, 1, -1):
        live = np.flatnonzero(alive)
        first = live[np.argmin(rank[live])]
        added = np.zeros(n, dtype=bool)
        added[first] = True
        tight = w[first].copy()
        before, last, phase_cut = first, first, 0.0
        for _ in range(remaining - 1):
            open_ = alive & ~added
            scores = np.where(open_, tight, -np.inf)
            hi = scores.max()
            cands = np.flatnonzero(open_ & (scores == hi))
            pick = cands[np.argmin(rank[cands])]
            phase_cut = tight[pick]
            before, last = last, pick
            added[pick] = True
            tight += w[pick]
        if phase_cut < best_w:
            best_w, best_side = float(phase_cut), list(members[last])
        # contract `last` into `before`
        w[before, :] += w[last, :]
        w[before, before] = 0.0
        w[before, last] = 0.0
        w[:, before] = w[before, :]
        alive[last] = False
        members[before].extend(members[last])
        rank[before] = min(rank[before], rank[last])
    return float(best_w), sorted(best_side)


def component_min_2cut(graph: ClusterGraph, comp: Tuple[int, ...]):
    """(weight, side slots, rest slots) of the induced subgraph on ``comp``."""
    sub = graph.weights[np.ix_(comp, comp)]
    weight, side_local = min_cut_kernel(sub, graph._lexrank[list(comp)])
    side = tuple(comp[i] for i in side_local)
    on_side = set(side)
    return weight, side, tuple(i for i in comp if i not in on_side)


def split_min_k_cut_sequence(graph: ClusterGraph, k_max: int) -> List[Partition]:
    """Partitions for k = 1..k_max by repeatedly removing the cheapest min 2-cut
    among the current components (ties: component with the smallest id)."""
    n = len(graph)
    if not 1 <= k_max <= n:
        raise PartitionError(f"k_max must be in 1..{n}, got {k_max}")
    comps: List[Tuple[int, ...]] = [tuple(range(n))]
    memo: Dict[Tuple[int, ...], tuple] = {}

    def current():
        return [frozenset(graph.vertices[i] for i in c) for c in comps]

    out = [make_partition(graph, current())]
    for _ in range(k_max - 1):
        choice, key = None, None
        for c in comps:
            if len(c) < 2:
                continue
            if c not in memo:
                memo[c] = component_min_2cut(graph, c)
            k = (memo[c][0], min(graph.vertices[i] for i in c))
            if key is None or k < key:
                key, choice = k, c
        if choice is None:
            raise PartitionError("no splittable component left")
        _, side, rest = memo[choice]
        comps.remove(choice)
        comps.extend([side, rest])
        out.append(make_partition(graph, current()))
    return out
