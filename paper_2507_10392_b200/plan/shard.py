"""Uneven, compute-proportional ZeRO-3 shard layout (new contract).

The reference shards every layer evenly (``/ d_dp`` at costs.py:262, 589, 592
and simulate.py:217, 450, 547, 577-585).  On B200 each DP-group member owns a
contiguous slice of every flat parameter buffer whose size is proportional to
its microbatch share, so Adam work, optimizer memory and RS/AG receive volume
track the planner's compute split.  Integer-only and deterministic:

    units      = ceil(P / A)                      (A = 64 elements, 128 B of bf16)
    counts     = proportional_split(units, shares, min_each=1)   (configure.py:311)
    [lo, hi)_r = cumulative counts * A, the last rank clipped to P

``min_each=1`` keeps a zero-share device in every collective with a non-empty
shard (the reference keeps zero-share devices in collectives: simulate.py:351-357).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

from .configure import TrainingPlan, proportional_split

SHARD_ALIGN = 64


@dataclass(frozen=True)
class ShardSpec:
    """Shard boundaries of one flat buffer of ``numel`` elements over a group."""

    numel: int
    bounds: Tuple[Tuple[int, int], ...]  # per device, in group device order

    @property
    def counts(self) -> List[int]:
        return [hi - lo for lo, hi in self.bounds]

    @property
    def displs(self) -> List[int]:
        return [lo for lo, _ in self.bounds]


def split_flat(numel: int, shares: Sequence[int], align: int = SHARD_ALIGN) -> ShardSpec:
    g = len(shares)
    units = -(-numel // align)
    if units < g:
        raise ValueError(f"buffer of {numel} elements is too small to shard over {g} ranks")
    counts = proportional_split(units, [float(s) for s in shares], min_each=1)
    bounds, lo = [], 0
    for c in counts:
        hi = min(lo + c * align, numel)
        bounds.append((lo, hi))
        lo = hi
    return ShardSpec(numel=numel, bounds=tuple(bounds))


def shard_layout(plan: TrainingPlan, params_of) -> Dict[int, Dict[int, ShardSpec]]:
    """{group index: {model layer: ShardSpec}} for every layer of every group.

    ``params_of(layer)`` gives the layer's parameter count (``ModelSpec.params_of``).
    """
    ranges = plan.stage_layer_ranges()
    out: Dict[int, Dict[int, ShardSpec]] = {gi: {} for gi in range(len(plan.groups))}
    for (gi, _), (lo, hi) in zip(plan.global_order(), ranges):
        g = plan.groups[gi]
        shares = [g.shares[d] for d in g.device_ids]
        for layer in range(lo, hi):
            out[gi][layer] = split_flat(params_of(layer), shares)
    return out
