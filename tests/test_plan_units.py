"""Known-answer tests for the planner heuristics, taken from the reference's own
tests (hetplan tests/test_configure.py, tests/test_costs.py)."""

import itertools
import random

import pytest

from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan.configure import GpuGroup, TrainingPlan
from paper_2507_10392_b200.plan.workload import GpuDevice, LayerFit, LayerRuntimeModel


def dev(i, kind="a100", node="n0"):
    return GpuDevice(id=f"{kind}-{i}", kind=kind, peak_tflops=100.0, mem_capacity=16_000_000_000,
                     node_id=node, region_id="r0")


def test_proportional_split_goldens():  # test_configure.py:46-58
    assert P.proportional_split(20, [2, 2, 1]) == [8, 8, 4]
    assert P.proportional_split(20, [1, 1, 1]) == [7, 7, 6]
    assert P.proportional_split(20, [2, 2, 1], min_each=1) == [8, 8, 4]
    assert P.proportional_split(5, [100, 1, 1], min_each=1) == [3, 1, 1]
    assert P.proportional_split(9, [0, 0, 0]) == [3, 3, 3]
    with pytest.raises(ValueError):
        P.proportional_split(2, [1, 1, 1], min_each=1)
    with pytest.raises(ValueError):
        P.proportional_split(5, [])
    with pytest.raises(ValueError):
        P.proportional_split(5, [1, -1])


def test_proportional_split_monotone():  # test_configure.py:60-71
    rng = random.Random(7)
    for _ in range(200):
        n = rng.randint(2, 6)
        w = [rng.uniform(0.1, 10.0) for _ in range(n)]
        total = rng.randint(n, 40)
        out = P.proportional_split(total, w, min_each=1)
        assert sum(out) == total
        for i in range(n):
            for j in range(n):
                if w[i] >= w[j]:
                    assert out[i] >= out[j] or w[i] == w[j]


def test_partition_layers_and_ministages():  # test_configure.py:82-106
    assert P.partition_layers([2.0, 2.0, 1.0], 20) == [8, 8, 4]
    assert P.partition_layers([100.0, 1.0], 2) == [1, 1]
    assert P.make_ministages(8, 4) == (2, 2, 2, 2)
    assert P.make_ministages(5, 2) == (3, 2)
    assert P.make_ministages(7, 3) == (3, 2, 2)
    assert P.make_ministages(5, 1) == (5,)
    assert P.make_ministages(5, 5) == (1, 1, 1, 1, 1)
    for bad in ((3, 4), (3, 0)):
        with pytest.raises(ValueError):
            P.make_ministages(*bad)


def _group(devs, bw):
    return GpuGroup(devices=tuple(devs), layers_assigned=1, ministage_sizes=(1,),
                    shares={d.id: 1 for d in devs}, aggregate_speed=1.0, intra_bw=bw)


def test_order_groups():  # test_configure.py:117-131
    a = _group([dev(0), dev(1)], 10e9)
    b = _group([dev(2, node="n1"), dev(3, node="n1")], 25e9)
    assert P.order_groups([a, b]) == [b, a]
    a = _group([dev(0), dev(1)], 25e9)
    b = _group([dev(5)], float("inf"))
    assert P.order_groups([a, b]) == [b, a]
    a = _group([dev(3)], float("inf"))
    b = _group([dev(1)], float("inf"))
    assert P.order_groups([a, b]) == [b, a]


def test_balance_microbatch_two_to_one():  # test_configure.py:135-141
    devs = [dev(0, "fast"), dev(1, "slow")]
    rt = LayerRuntimeModel(fits={("fast", "transformer"): LayerFit(0.0, 0.002, 0.0, 0.004),
                                 ("slow", "transformer"): LayerFit(0.0, 0.004, 0.0, 0.008)})
    assert P.balance_microbatch(devs, rt, 12) == {"fast-0": 8, "slow-1": 4}


def test_balance_microbatch_exhaustive_minimax():  # test_configure.py:150-188
    rng = random.Random(11)
    for trial in range(40):
        n = rng.randint(2, 3)
        fits = {}
        devs = []
        for i in range(n):
            k = f"k{trial}_{i}"
            fits[(k, "transformer")] = LayerFit(rng.uniform(0, .002), rng.uniform(.001, .01),
                                                rng.uniform(0, .004), rng.uniform(.002, .02))
            devs.append(GpuDevice(id=f"d{i}", kind=k, peak_tflops=1.0, mem_capacity=1,
                                  node_id="n0", region_id="r0"))
        rt = LayerRuntimeModel(fits=fits)
        size = rng.randint(1, 12)

        def t(i, s):
            f = fits[(devs[i].kind, "transformer")]
            return 0.0 if s <= 0 else f.fwd_alpha + f.bwd_alpha + (f.fwd_beta + f.bwd_beta) * s

        best = min(max(t(i, c[i]) for i in range(n))
                   for c in itertools.product(range(size + 1), repeat=n) if sum(c) == size)
        shares = P.balance_microbatch(devs, rt, size)
        assert sum(shares.values()) == size
        assert max(t(i, shares[f"d{i}"]) for i in range(n)) == pytest.approx(best, rel=1e-9)


def test_route_microbatches():  # test_configure.py:197-229
    routed = P.route_microbatches({"a": 2, "b": 1}, 3, {"a": 1.0, "b": 2.0})
    assert len(routed) == 3 and all(sorted(mb) == [("a", 2), ("b", 1)] for mb in routed)
    assert P.route_microbatches({"a": 1, "b": 1}, 2, {"a": 5.0, "b": 1.0})[0][0][0] == "a"
    assert all(mb == [("a", 3)] for mb in P.route_microbatches({"a": 3, "b": 0}, 2,
                                                                 {"a": 1.0, "b": 1.0}))


def _geo_plan(sizes_per_group):
    groups = []
    for gi, sizes in enumerate(sizes_per_group):
        d = (dev(gi * 10, node=f"n{gi}"),)
        groups.append(GpuGroup(devices=d, layers_assigned=sum(sizes), ministage_sizes=tuple(sizes),
                               shares={d[0].id: 4}, aggregate_speed=1.0, intra_bw=float("inf")))
    return TrainingPlan(groups=tuple(groups), n_microbatches=2, microbatch_size=4,
                        strategy=P.Strategy.INTERLEAVED, cluster_fingerprint="x")


def test_global_order_and_ranges():  # test_configure.py:246-256
    assert _geo_plan([(2, 2), (3, 3)]).global_order() == [(0, 0), (1, 0), (0, 1), (1, 1)]
    assert _geo_plan([(2, 2, 2), (5,)]).global_order() == [(0, 0), (1, 0), (0, 1), (0, 2)]
    assert _geo_plan([(2, 2), (3, 3)]).stage_layer_ranges() == [(0, 2), (2, 5), (5, 7), (7, 10)]


def test_plan_validation():  # test_configure.py:258-276
    with pytest.raises(P.PlanFormatError):
        d = (dev(0),)
        TrainingPlan(groups=(GpuGroup(devices=d, layers_assigned=2, ministage_sizes=(2,),
                                      shares={d[0].id: 3}, aggregate_speed=1.0,
                                      intra_bw=float("inf")),),
                     n_microbatches=2, microbatch_size=4, strategy=P.Strategy.INTERLEAVED,
                     cluster_fingerprint="x")
    with pytest.raises(P.PlanFormatError):
        GpuGroup(devices=(dev(0),), layers_assigned=5, ministage_sizes=(2, 2),
                 shares={"a100-0": 1}, aggregate_speed=1.0, intra_bw=1e9)


def test_count_collectives():  # test_costs.py:171-181
    assert P.count_collectives(20, 3, P.Strategy.INTERLEAVED) == (40, 20)
    assert P.count_collectives(20, 3, P.Strategy.PP_ZERO2) == (40, 20)
    assert P.count_collectives(20, 3, P.Strategy.PP_ZERO3) == (120, 20)


def test_split_flat_edges():
    s = P.split_flat(7_087_872, [11, 11, 11, 11, 5, 5, 5, 5])
    assert s.counts == [1_218_176] * 4 + [553_792] * 4   # SURVEY §8 a12 worked example
    s = P.split_flat(1000, [0, 0, 0])                     # zero shares -> even, non-empty
    assert s.counts == [384, 320, 296]
    s = P.split_flat(1000, [8, 0])                        # zero-share rank keeps one unit
    assert s.counts == [960, 40]
    with pytest.raises(ValueError):
        P.split_flat(64, [1, 1])                          # fewer 64-element units than ranks


def test_native_min_cut_matches_numpy_twin():
    """zb_min_cut (csrc/mincut.cpp, the native twin of the reference's compiled
    min_cut_kernel) is bit-identical to the numpy restatement, ties included."""
    import numpy as np
    from paper_2507_10392_b200.plan import mincut as MC
    if MC.native_kernel() is None:
        pytest.skip("library not built")
    rng = np.random.default_rng(7)
    for trial in range(200):
        n = int(rng.integers(2, 14))
        if trial % 3 == 0:   # integer weights: many ties
            w = rng.integers(0, 4, size=(n, n)).astype(np.float64)
        else:
            w = rng.random((n, n)) * rng.choice([1.0, 1e-3, 1e6])
        w = np.triu(w, 1)
        w = w + w.T
        rank = rng.permutation(n).astype(np.int64)
        assert MC.min_cut_native(w, rank) == MC.min_cut_python(w, rank), trial


def test_native_eq1_latency_bit_identical():
    """zb_eq1_latency (csrc/eq1.cpp) equals the Python Eq.1 restatement bit for bit on
    every golden plan (reference layouts, searches, the reference's agreement suite)."""
    import json
    import os
    from paper_2507_10392_b200.plan import estimate as ES
    if ES._native_eq1() is None:
        pytest.skip("library not built")
    gold = os.path.join(os.path.dirname(__file__), "golden")
    cases = json.load(open(os.path.join(gold, "plans.json")))
    checked = 0
    for case in cases:
        prof = P.load_cluster_profile(os.path.join(gold, case["cluster"]))
        model, workload = P.load_model_workload(os.path.join(gold, case["model"]))
        ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=P.fit_runtime_model(prof),
                            model=model, workload=workload)
        plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
        for strat in (P.Strategy.INTERLEAVED, P.Strategy.PP_ZERO2, P.Strategy.PP_ZERO3):
            plan.strategy = strat
            a = ES.total_iteration_latency(ctx, plan)
            b = ES.total_iteration_latency_py(ctx, plan)
            assert (a.l_forwards, a.l_backwards, a.l_startup) == \
                (b.l_forwards, b.l_backwards, b.l_startup), (case["name"], strat)
            checked += 1
    assert checked == 3 * len(cases)
