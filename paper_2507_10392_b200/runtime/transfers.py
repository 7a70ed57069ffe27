"""Sample dealing and stage-boundary transfer lists (pure host logic).

Microbatch m covers global samples [m*mbs, (m+1)*mbs); inside group G they are
dealt contiguously to devices in ``routing[G][m]`` order (configure.py:414-430).
A boundary between adjacent global stages held by different groups moves every
sample of the microbatch from the device that holds it in the sending group to
the device that holds it in the receiving group: the transfer set is the interval
intersections of the two groups' sample ranges.  The reference ships a boundary
over one best link (simulate.py:378-385, 507-514; boundary bytes :274-277); the
total bytes and the event count are the same, only the per-pair split is new.
"""

from __future__ import annotations

from typing import Dict, List, Tuple


def sample_ranges(plan) -> List[List[Dict[str, Tuple[int, int]]]]:
    """ranges[gi][m][dev] = (lo, hi) sample offsets inside microbatch m."""
    out = []
    mbs = plan.microbatch_size
    for gi, g in enumerate(plan.groups):
        per_m = []
        for m in range(plan.n_microbatches):
            off, r = 0, {}
            for dev, cnt in plan.routing[gi][m]:
                r[dev] = (off, off + cnt)
                off += cnt
            if off != mbs:
                raise ValueError(f"routing of group {gi} microbatch {m} covers {off} samples")
            for dev in g.device_ids:
                r.setdefault(dev, (0, 0))
            per_m.append(r)
        out.append(per_m)
    return out


def pair_intersections(plan, ranges, g_from: int, g_to: int, m: int):
    """(src dev, dst dev, sample lo, sample hi) intersections for microbatch m."""
    src, dst = ranges[g_from][m], ranges[g_to][m]
    out = []
    for a in plan.groups[g_from].device_ids:
        alo, ahi = src[a]
        for b in plan.groups[g_to].device_ids:
            blo, bhi = dst[b]
            lo, hi = max(alo, blo), min(ahi, bhi)
            if lo < hi:
                out.append((a, b, lo, hi))
    return out


def boundary_transfers(plan, ranges, dev_id: str, rank_of: Dict[str, int], seq_len: int):
    """Per (direction "f"|"b", boundary s, microbatch m): this device's list of
    (peer world rank, row lo, row hi, is_send); rows index its [share*S, d] buffer.
    Forward sends the output of stage s (group of s -> group of s+1), backward the
    gradient of stage s+1's input (the other way)."""
    order = plan.global_order()
    out = {}
    for s in range(len(order) - 1):
        ga, gb = order[s][0], order[s + 1][0]
        if ga == gb:
            continue
        for m in range(plan.n_microbatches):
            for direction, (g_from, g_to) in (("f", (ga, gb)), ("b", (gb, ga))):
                lst = []
                for a, b, lo, hi in pair_intersections(plan, ranges, g_from, g_to, m):
                    if a == dev_id:
                        base = ranges[g_from][m][dev_id][0]
                        lst.append((rank_of[b], (lo - base) * seq_len, (hi - base) * seq_len, True))
                    if b == dev_id:
                        base = ranges[g_to][m][dev_id][0]
                        lst.append((rank_of[a], (lo - base) * seq_len, (hi - base) * seq_len, False))
                out[(direction, s, m)] = lst
    return out
