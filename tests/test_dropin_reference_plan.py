"""Drop-in check: a plan object produced by the UNMODIFIED reference planner
(hetplan, imported from /root/reference in the build container) runs through
the executor unchanged — same TrainingPlan / CostContext objects the
reference's simulate_plan(ctx, plan) consumes (simulate.py:590).  Host logic on
CPU (test-only kernel twin); skipped where the reference is not mounted."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def test_reference_plan_objects_execute_and_match_oracle(monkeypatch):
    monkeypatch.syspath_prepend(REF)
    monkeypatch.setenv("HETPLAN_PURE_PYTHON", "1")
    import cpu_ops
    import hetplan
    from hetplan import configure as rc
    from hetplan.costs import CostContext, Strategy
    from hetplan.partition import build_cluster_graph, make_partition
    from hetplan.workload import ClusterProfile, GpuDevice, ModelSpec, WorkloadSpec, fit_runtime_model

    from oracle import gpt_cpu
    from paper_2507_10392_b200.plan import emulated as E
    from paper_2507_10392_b200.runtime.data import synthetic_batch
    from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

    cfg = E.ModelConfig("ref-dropin", "gpt", n_layer=2, d_model=64, n_head=2, vocab=256, seq_len=64)
    raw = E.profile_json([("n0", ["b200"])])
    prof = ClusterProfile(
        devices=tuple(GpuDevice(**{k: e[k] for k in ("id", "kind", "peak_tflops", "mem_capacity",
                                                      "node_id", "region_id")})
                      for e in raw["devices"]),
        intra_node_bw=raw["intra_node_bw"], inter_node_bw={},
        runtime_samples={(k, c): [tuple(s) for s in series]
                         for k, per in raw["runtime_samples"].items() for c, series in per.items()})
    rt = fit_runtime_model(prof)
    graph = build_cluster_graph(prof)
    ctx = CostContext(graph=graph, runtime=rt,
                      model=ModelSpec.uniform(cfg.n_layer, cfg.params_per_layer(), cfg.d_model, 2),
                      workload=WorkloadSpec(4, cfg.seq_len))
    plan = rc.build_plan(ctx, prof, make_partition(graph, [frozenset(["n0-0"])]), 2, [2],
                         Strategy.INTERLEAVED, rc.cluster_fingerprint(prof), "transformer")
    plan.routing = [rc.route_microbatches(g.shares, plan.n_microbatches,
                                          {d.id: rc._per_sample_time(rt, d, "transformer")
                                           for d in g.devices}) for g in plan.groups]
    assert type(plan).__module__ == "hetplan.configure"      # the reference's own object
    tr = ZorseTrainer(plan, ctx, cfg, _ops=cpu_ops)
    batch = synthetic_batch(cfg.vocab, cfg.seq_len, 4, 1)
    loss = tr.step(batch)
    ref, _ = gpt_cpu.loss_and_grads(cfg, gpt_cpu.init_params(cfg, 1234), batch)
    assert abs(loss - ref) / ref < 1e-2
    # the executor's instruction stream is the reference simulator's event order
    from hetplan.simulate import simulate_plan
    tl = simulate_plan(ctx, plan)
    ours = [(e.kind, e.stage, e.microbatch, e.layer) for e in tr.exec.events]
    assert ours == [(e.kind, e.stage, e.microbatch, e.layer) for e in tl.events]
