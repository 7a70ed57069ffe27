"""Generate golden plan / schedule / shard fixtures from the REFERENCE (hetplan).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src HETPLAN_PURE_PYTHON=1 python tests/golden/make_golden.py

It imports the unmodified reference planner and simulator from
/root/reference/pkg/src and records, for each BASELINE layout and for a
randomized slice of the reference's own agreement suite (fixtures.py:213):

* the cluster profile / model JSON inputs (reference file formats),
* the plan file bytes (``TrainingPlan.save``) with routing attached
  (configure.py:700-707 / route_microbatches configure.py:414),
* the full simulated event order (simulate.py:590-649) with exact float reprs,
* per-group collective counts,
* shard boundaries computed with the reference ``proportional_split``.

The product restatement (paper_2507_10392_b200.plan) is checked against these
files by tests/test_plan_parity.py.
"""

from __future__ import annotations

import io
import json
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import hetplan  # noqa: E402  (reference)
from hetplan import configure as rc  # noqa: E402
from hetplan import fixtures as rf  # noqa: E402
from hetplan.costs import CostContext, Strategy  # noqa: E402
from hetplan.partition import build_cluster_graph, make_partition, split_min_k_cut_sequence  # noqa: E402
from hetplan.simulate import simulate_plan  # noqa: E402
from hetplan.workload import fit_runtime_model, load_cluster_profile, load_model_workload  # noqa: E402

from paper_2507_10392_b200.plan import emulated as E  # noqa: E402  (only for the input JSON)


def _dump(obj, name):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)
        fh.write("\n")


def _events(tl):
    return [[e.kind, e.group, e.stage, e.microbatch, e.layer, repr(e.start), repr(e.end),
             list(e.device_ids), e.lane] for e in tl.events]


def _plan_text(plan):
    buf = io.StringIO()
    json.dump(plan.to_json_dict(), buf, indent=2, sort_keys=True)
    buf.write("\n")
    return buf.getvalue()


def _ref_shards(plan, params_of, align=64):
    """Uneven shard rule evaluated with the REFERENCE proportional_split."""
    out = {}
    for (gi, _), (lo, hi) in zip(plan.global_order(), plan.stage_layer_ranges()):
        g = plan.groups[gi]
        shares = [float(g.shares[d]) for d in g.device_ids]
        for layer in range(lo, hi):
            p = params_of(layer)
            counts = rc.proportional_split(-(-p // align), shares, min_each=1)
            b, c = [], 0
            for n in counts:
                e = min(c + n * align, p)
                b.append([c, e])
                c = e
            out[str(layer)] = b
    return out


def fixed_layout_case(name, nodes, model_cfg, global_batch, groups, n_mb, counts, strategy):
    prof_json = E.profile_json(nodes)
    model_json = model_cfg.model_json(global_batch)
    pf = os.path.join(HERE, f"cluster_{name}.json")
    mf = os.path.join(HERE, f"model_{name}.json")
    _dump(prof_json, f"cluster_{name}.json")
    _dump(model_json, f"model_{name}.json")
    profile = load_cluster_profile(pf)
    model, workload = load_model_workload(mf)
    runtime = fit_runtime_model(profile)
    graph = build_cluster_graph(profile)
    ctx = CostContext(graph=graph, runtime=runtime, model=model, workload=workload)
    part = make_partition(graph, [frozenset(g) for g in groups])
    plan = rc.build_plan(ctx, profile, part, n_mb, counts, Strategy(strategy),
                         rc.cluster_fingerprint(profile), "transformer")
    plan.routing = [rc.route_microbatches(
        g.shares, plan.n_microbatches,
        {d.id: rc._per_sample_time(runtime, d, "transformer") for d in g.devices})
        for g in plan.groups]
    tl = simulate_plan(ctx, plan)
    return {
        "name": name, "kind": "build_plan", "cluster": f"cluster_{name}.json",
        "model": f"model_{name}.json", "groups": [sorted(g) for g in groups],
        "n_microbatches": n_mb, "ministage_counts": list(counts), "strategy": strategy,
        "plan_json": _plan_text(plan), "events": _events(tl),
        "iteration_time": repr(tl.iteration_time),
        "collective_counts": {str(k): v for k, v in tl.collective_counts.items()},
        "global_order": [list(x) for x in plan.global_order()],
        "stage_layer_ranges": [list(x) for x in plan.stage_layer_ranges()],
        "shards": _ref_shards(plan, model.params_of),
    }


def planner_case(name, nodes, model_cfg, global_batch, k_max=None, strategies=("zorse",),
                 prof_json=None):
    prof_json = prof_json if prof_json is not None else E.profile_json(nodes)
    _dump(prof_json, f"cluster_{name}.json")
    _dump(model_cfg.model_json(global_batch), f"model_{name}.json")
    profile = load_cluster_profile(os.path.join(HERE, f"cluster_{name}.json"))
    model, workload = load_model_workload(os.path.join(HERE, f"model_{name}.json"))
    runtime = fit_runtime_model(profile)
    plan, records = rc.plan_training(profile, model, workload, runtime,
                                     strategies=tuple(Strategy(s) for s in strategies), k_max=k_max)
    ctx = CostContext(graph=build_cluster_graph(profile), runtime=runtime, model=model,
                      workload=workload)
    tl = simulate_plan(ctx, plan)
    return {
        "name": name, "kind": "plan_training", "cluster": f"cluster_{name}.json",
        "model": f"model_{name}.json", "k_max": k_max, "strategies": list(strategies),
        "n_candidates": len(records), "plan_json": _plan_text(plan), "events": _events(tl),
        "iteration_time": repr(tl.iteration_time),
        "collective_counts": {str(k): v for k, v in tl.collective_counts.items()},
        "shards": _ref_shards(plan, model.params_of),
    }


def measured_profile_case(name, profile_path, model_cfg, global_batch, k_max=None):
    """plan_training on a cluster profile whose runtime samples were MEASURED on B200
    (scripts/profile_layers.py; the planner loop closed on real layer timings)."""
    with open(os.path.join(ROOT, profile_path)) as fh:
        raw = json.load(fh)
    return planner_case(name, None, model_cfg, global_batch, k_max=k_max,
                        prof_json=raw.get("cluster_profile", raw))


def reference_fixture_case(name, profile, model, workload, **kw):
    """plan_training on one of the reference's own fixture clusters."""
    _dump(rf.profile_to_json_dict(profile), f"cluster_{name}.json")
    _dump(rf.model_to_json_dict(model, workload), f"model_{name}.json")
    prof = load_cluster_profile(os.path.join(HERE, f"cluster_{name}.json"))
    m, w = load_model_workload(os.path.join(HERE, f"model_{name}.json"))
    runtime = fit_runtime_model(prof)
    plan, records = rc.plan_training(prof, m, w, runtime, **kw)
    return {"name": name, "kind": "plan_training", "cluster": f"cluster_{name}.json",
            "model": f"model_{name}.json", "k_max": kw.get("k_max"), "strategies": ["zorse"],
            "n_candidates": len(records), "plan_json": _plan_text(plan), "events": None,
            "shards": None}


def agreement_cases(seed, n):
    """Randomized feasible plans from the reference's own suite, serialized."""
    out = []
    for i, (ctx, plan) in enumerate(rf.agreement_suite(seed, n)):
        # recover the profile from the graph's devices: the suite cycles 3 fixtures
        profile = [rf.toy_cluster(), rf.slow_interconnect_cluster(), rf.two_region_cluster()][i % 3]
        tl = simulate_plan(ctx, plan)
        out.append({
            "cluster": rf.profile_to_json_dict(profile),
            "model": rf.model_to_json_dict(ctx.model, ctx.workload),
            "plan_json": _plan_text(plan),
            "events": _events(tl),
            "collective_counts": {str(k): v for k, v in tl.collective_counts.items()},
        })
    return out


def main():
    cases = [
        fixed_layout_case("tiny", E.CONFIG_NODES["tiny-2stage"], E.TINY_GPT, 8,
                          [["n0-0", "n0-1"], ["n1-0"]], 2, [1, 1], "zorse"),
        fixed_layout_case("tiny_ms", E.CONFIG_NODES["tiny-2stage"], E.TINY_GPT, 8,
                          [["n0-0", "n0-1"], ["n1-0"]], 2, [2, 2], "zorse"),
        fixed_layout_case("tiny_z3", E.CONFIG_NODES["tiny-2stage"], E.TINY_GPT, 8,
                          [["n0-0", "n0-1"], ["n1-0"]], 2, [1, 2], "pp-zero3"),
        fixed_layout_case("gpt2s_dp8", E.dp_group_nodes(8), E.GPT2_SMALL, 64,
                          [[f"n0-{i}" for i in range(8)]], 1, [12], "zorse"),
        fixed_layout_case("gpt2s_dp4", E.dp_group_nodes(4), E.GPT2_SMALL, 32,
                          [[f"n0-{i}" for i in range(4)]], 1, [12], "zorse"),
        fixed_layout_case("gpt2s_dp2", E.dp_group_nodes(2), E.GPT2_SMALL, 16,
                          [[f"n0-{i}" for i in range(2)]], 1, [12], "zorse"),
        fixed_layout_case("gpt2s_dp1", E.dp_group_nodes(1), E.GPT2_SMALL, 8,
                          [["n0-0"]], 1, [12], "zorse"),
        fixed_layout_case("xl_3p5", E.CONFIG_NODES["xl-3+5"], E.GPT2_XL, 64,
                          [["n0-0", "n0-1", "n0-2"], [f"n1-{i}" for i in range(5)]], 8, [1, 1],
                          "zorse"),
        fixed_layout_case("llama7b_4x2", E.CONFIG_NODES["llama7b-4x2"], E.LLAMA_7B, 32,
                          [[f"n{i}-0", f"n{i}-1"] for i in range(4)], 8, [1, 1, 1, 1], "pp-zero3"),
        planner_case("tiny_search", E.CONFIG_NODES["tiny-2stage"], E.TINY_GPT, 8, k_max=2),
        planner_case("gpt2s_search", E.dp_group_nodes(8), E.GPT2_SMALL, 64, k_max=1),
        planner_case("llama13b_search", E.CONFIG_NODES["llama13b-8"], E.LLAMA_13B, 256),
        measured_profile_case("gpt2s_measured8", "profiles/r01_measured_b200_profile_gpt2s.json",
                              E.GPT2_SMALL, 64, k_max=1),
        # the reference README's planner benchmark: 128 GPUs, ~1,600 candidates (README:139-140)
        reference_fixture_case("ref_128gpu", rf.large_two_region_cluster(), rf.transformer_model(),
                               rf.default_workload()),
    ]
    _dump(cases, "plans.json")
    _dump(agreement_cases(seed=2024, n=12), "agreement.json")
    print(f"wrote {len(cases)} layout cases and agreement suite via hetplan {hetplan.__version__}")


if __name__ == "__main__":
    main()
