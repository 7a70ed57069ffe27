"""Plan / schedule / shard parity with the reference (hetplan), CPU only.

Golden files come from tests/golden/make_golden.py, which runs the unmodified
reference.  Everything here must match bit for bit: plan-file bytes, routing,
global ministage order, layer ranges, the full simulated event order (kinds,
groups, stages, microbatches, layers, devices, lanes and float start/end
times), collective counts and shard boundaries.
"""

import json
import os

import pytest

from paper_2507_10392_b200 import plan as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


CASES = _load("plans.json")


def _ctx(case):
    prof = P.load_cluster_profile(os.path.join(GOLD, case["cluster"]))
    model, workload = P.load_model_workload(os.path.join(GOLD, case["model"]))
    rt = P.fit_runtime_model(prof)
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=model,
                        workload=workload)
    return prof, ctx


def _events(sched):
    return [[e.kind, e.group, e.stage, e.microbatch, e.layer, repr(e.start), repr(e.end),
             list(e.device_ids), e.lane] for e in sched.events]


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "build_plan"],
                         ids=lambda c: c["name"])
def test_build_plan_bit_exact(case):
    prof, ctx = _ctx(case)
    part = P.make_partition(ctx.graph, case["groups"])
    plan = P.build_plan(ctx, prof, part, case["n_microbatches"], case["ministage_counts"],
                        P.Strategy(case["strategy"]), P.cluster_fingerprint(prof), "transformer")
    P.attach_routing(plan, ctx.runtime, "transformer")
    assert plan.dumps() == case["plan_json"]
    assert [list(x) for x in plan.global_order()] == case["global_order"]
    assert [list(x) for x in plan.stage_layer_ranges()] == case["stage_layer_ranges"]


@pytest.mark.parametrize("case", [c for c in CASES if c["events"] is not None],
                         ids=lambda c: c["name"])
def test_schedule_bit_exact(case):
    prof, ctx = _ctx(case)
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    # load/save round trip preserves every value (ints in planner-emitted memory
    # estimates come back as floats, exactly as with the reference's own loader)
    assert json.loads(plan.dumps()) == json.loads(case["plan_json"])
    sched = P.build_schedule(ctx, plan)
    assert _events(sched) == case["events"]
    assert repr(sched.iteration_time) == case["iteration_time"]
    counts = {str(k): v for k, v in sched.collective_counts().items()}
    assert counts == case["collective_counts"]
    for gi, g in enumerate(plan.groups):
        ag, rs = P.count_collectives(g.layers_assigned, plan.n_microbatches, plan.strategy)
        assert counts[str(gi)] == {"allgather": ag, "reduce_scatter": rs}


@pytest.mark.parametrize("case", [c for c in CASES if c["shards"] is not None],
                         ids=lambda c: c["name"])
def test_shard_layout_matches_reference_apportionment(case):
    prof, ctx = _ctx(case)
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    layout = P.shard_layout(plan, ctx.model.params_of)
    got = {str(layer): [list(b) for b in spec.bounds]
           for per_group in layout.values() for layer, spec in per_group.items()}
    assert got == case["shards"]
    for per_group in layout.values():
        for layer, spec in per_group.items():
            assert spec.bounds[0][0] == 0 and spec.bounds[-1][1] == ctx.model.params_of(layer)
            assert all(a[1] == b[0] for a, b in zip(spec.bounds, spec.bounds[1:]))
            assert all(lo % 64 == 0 for lo, _ in spec.bounds)


AGREEMENT = _load("agreement.json")


@pytest.mark.parametrize("idx", range(len(AGREEMENT)))
def test_agreement_suite_schedules(idx, tmp_path):
    case = AGREEMENT[idx]
    pf, mf = tmp_path / "c.json", tmp_path / "m.json"
    pf.write_text(json.dumps(case["cluster"]))
    mf.write_text(json.dumps(case["model"]))
    prof = P.load_cluster_profile(str(pf))
    model, workload = P.load_model_workload(str(mf))
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=P.fit_runtime_model(prof),
                        model=model, workload=workload)
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    assert json.loads(plan.dumps()) == json.loads(case["plan_json"])
    sched = P.build_schedule(ctx, plan)
    assert _events(sched) == case["events"]
    assert {str(k): v for k, v in sched.collective_counts().items()} == case["collective_counts"]


def test_device_streams_partition_the_events():
    case = next(c for c in CASES if c["name"] == "xl_3p5")
    prof, ctx = _ctx(case)
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    sched = P.build_schedule(ctx, plan)
    order = plan.global_order()
    seen = set()
    for gi, g in enumerate(plan.groups):
        streams = [sched.stream_for(d) for d in g.device_ids]
        assert all(s == streams[0] for s in streams)  # group members run one program
        for e in streams[0]:
            if e.group != gi:  # only the receiving side of a boundary transfer
                peer = e.key[1] + 1 if e.key[0] == "PSf" else e.key[1]
                assert e.kind == "P2PSend" and order[peer][0] == gi
        seen |= {e.key for e in streams[0]}
        # streams keep the global order
        pos = {e.key: i for i, e in enumerate(sched.events)}
        idx = [pos[e.key] for e in streams[0]]
        assert idx == sorted(idx)
    assert seen == {e.key for e in sched.events}


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "plan_training"],
                         ids=lambda c: c["name"])
def test_plan_training_bit_exact(case):
    prof, ctx = _ctx(case)
    plan, records = P.plan_training(prof, ctx.model, ctx.workload, ctx.runtime,
                                    strategies=tuple(P.Strategy(s) for s in case["strategies"]),
                                    k_max=case["k_max"])
    assert len(records) == case["n_candidates"]
    assert plan.dumps() == case["plan_json"]


MEMORY = _load("memory.json")


@pytest.mark.parametrize("case", [c for c in CASES if c["name"] in MEMORY], ids=lambda c: c["name"])
def test_memory_replay_bit_exact(case, tmp_path):
    """The simulator's memory accounting (task effects, simulate.py:284-550; replay
    :660-696; initial residency :565-588) and its Gantt / memory CSV exports
    (:115-137), restated, reproduce the reference's peaks and file bytes."""
    import hashlib
    prof, ctx = _ctx(case)
    plan = P.TrainingPlan.from_json_dict(json.loads(case["plan_json"]), prof)
    sched = P.build_schedule(ctx, plan)
    peaks, traces = sched.memory(ctx)
    want = MEMORY[case["name"]]
    assert {d: {c: repr(v) for c, v in p.items()} for d, p in peaks.items()} == want["peaks"]
    from paper_2507_10392_b200.plan.schedule import write_gantt_csv, write_memory_csv
    write_gantt_csv(str(tmp_path / "g.csv"), sched.gantt_rows())
    write_memory_csv(str(tmp_path / "m.csv"), traces)
    sha = lambda p: hashlib.sha256(p.read_bytes()).hexdigest()  # noqa: E731
    assert sha(tmp_path / "g.csv") == want["gantt_sha256"]
    assert sha(tmp_path / "m.csv") == want["memory_sha256"]
