"""Stage-boundary transfer lists (runtime/transfers.py) against a brute-force
per-sample restatement, for every golden plan (tests/golden, made by the
unmodified reference planner).  CPU only.

Brute force: own[g][m][i] = the device of group g that holds sample i of
microbatch m (routing order, configure.py:414-430).  For each boundary between
stages of different groups, every sample must move exactly once from its owner in
the sending group to its owner in the receiving group, in both directions, and
the per-rank lists must be consistent (each send has the matching receive).  The
bytes per boundary and microbatch equal the reference's boundary volume
mb * s * d * 2 (simulate.py:274-277)."""

import json
import os
from collections import defaultdict

import pytest

from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.runtime.transfers import boundary_transfers, sample_ranges

GOLD = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLD, "plans.json")) as fh:
    CASES = json.load(fh)
S = 8   # rows per sample (any positive seq_len exercises the row arithmetic)


def _plan(case):
    prof = P.load_cluster_profile(os.path.join(GOLD, case["cluster"]))
    model, workload = P.load_model_workload(os.path.join(GOLD, case["model"]))
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    if plan.routing is None:
        P.attach_routing(plan, P.fit_runtime_model(prof), "transformer")
    return plan, [d.id for d in prof.devices]


def _owners(plan):
    own = []
    for gi in range(len(plan.groups)):
        per_m = []
        for m in range(plan.n_microbatches):
            seq = []
            for dev, cnt in plan.routing[gi][m]:
                seq += [dev] * cnt
            assert len(seq) == plan.microbatch_size
            per_m.append(seq)
        own.append(per_m)
    return own


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_boundary_transfers_match_brute_force(case):
    plan, devices = _plan(case)
    rank_of = {d: i for i, d in enumerate(devices)}
    ranges = sample_ranges(plan)
    own = _owners(plan)
    # sample ranges are the contiguous runs of the owner map
    for gi, per_m in enumerate(own):
        for m, seq in enumerate(per_m):
            for dev, (lo, hi) in ranges[gi][m].items():
                assert [i for i, o in enumerate(seq) if o == dev] == list(range(lo, hi))
    lists = {d: boundary_transfers(plan, ranges, d, rank_of, S) for d in devices
             if any(d in g.device_ids for g in plan.groups)}
    order = plan.global_order()
    for s in range(len(order) - 1):
        ga, gb = order[s][0], order[s + 1][0]
        if ga == gb:
            continue
        for m in range(plan.n_microbatches):
            for direction, (gf, gt) in (("f", (ga, gb)), ("b", (gb, ga))):
                # brute force: expected rows moved per (src, dst) pair
                want = defaultdict(int)
                for i in range(plan.microbatch_size):
                    want[(own[gf][m][i], own[gt][m][i])] += S
                sends, recvs = defaultdict(int), defaultdict(int)
                for dev, tl in lists.items():
                    for peer, lo, hi, is_send in tl[(direction, s, m)]:
                        assert 0 <= lo < hi
                        share = ranges[gf if is_send else gt][m][dev]
                        assert hi <= (share[1] - share[0]) * S   # inside this rank's rows
                        key = (dev, devices[peer]) if is_send else (devices[peer], dev)
                        (sends if is_send else recvs)[key] += hi - lo
                assert dict(sends) == dict(want)
                assert dict(recvs) == dict(want)
                assert sum(want.values()) == plan.microbatch_size * S


def _windows(case):
    from paper_2507_10392_b200.runtime.executor import WindowPlan
    plan, devices = _plan(case)
    prof = P.load_cluster_profile(os.path.join(GOLD, case["cluster"]))
    model, workload = P.load_model_workload(os.path.join(GOLD, case["model"]))
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=P.fit_runtime_model(prof),
                        model=model, workload=workload)
    sched = P.build_schedule(ctx, plan)
    order, ranges = plan.global_order(), plan.stage_layer_ranges()
    for gi, g in enumerate(plan.groups):
        mine = [s for s in range(len(order)) if order[s][0] == gi]
        chunks = {s: list(range(*ranges[s])) for s in mine}
        head = len(order) - 1 if order[-1][0] == gi else None
        plans = [WindowPlan(sched.stream_for(d), chunks, head, len(g.device_ids) > 1,
                            plan.strategy.gathers_per_microbatch) for d in g.device_ids]
        yield plan, gi, sched.stream_for(g.device_ids[0]), plans


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_window_slots(case):
    """Window-slot plans (runtime/executor.WindowPlan) for every golden plan: identical
    on every rank of a group (peers address each other's gradient slots by offset);
    INTERLEAVED materialises at most two ministages (simulate.py FREEf/FREEb ring,
    costs.py:566-571); at most two gradient slots; every slot handed over only after
    its previous holder's release event was issued earlier in the stream."""
    for plan, gi, events, plans in _windows(case):
        w = plans[0]
        for other in plans[1:]:
            assert (other.grad_slot, other.grad_prev, other.param_slot, other.param_prev) == \
                (w.grad_slot, w.grad_prev, w.param_slot, w.param_prev)
        assert w.n_grad_slots <= 2
        if plan.strategy.offloads and len(plan.groups[gi].device_ids) > 1:
            assert w.n_param_slots <= 2
        idx = {e.key: i for i, e in enumerate(events)}
        for s, (prev, same_step) in w.grad_prev.items():
            if prev is not None and same_step:
                head = s == len(plan.global_order()) - 1
                first = min(i for i, e in enumerate(events) if e.stage == s and
                            (e.kind == "Bwd" or (e.kind == "Fwd" and head)))
                last_rs = max(i for i, e in enumerate(events)
                              if e.kind == "ReduceScatter" and e.stage == prev)
                assert last_rs < first
        for key, prev in w.param_prev.items():
            if prev is not None:
                free = idx[("FREE" + prev[0], prev[1])]
                ag = idx[("AG" + key[0], key[1], 0)]
                assert free < ag
