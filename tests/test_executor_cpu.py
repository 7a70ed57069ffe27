"""Executor host logic on CPU: plan walking, uneven shards, routing, boundary
P2P and DP collectives (gloo, world_size 3), against the fp32 oracle.

The arithmetic is the test-only torch twin of the kernels (tests/cpu_ops.py),
so these tests pin the executor's data movement; the B200 kernels themselves
are pinned by the gpu-marked tests.
"""

import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import cpu_ops  # noqa: E402

from oracle import parity  # noqa: E402
from paper_2507_10392_b200 import plan as P  # noqa: E402
from paper_2507_10392_b200.plan import emulated as E  # noqa: E402
from paper_2507_10392_b200.runtime.data import synthetic_batch  # noqa: E402
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer  # noqa: E402

CFG = E.ModelConfig("tiny-test", "gpt", n_layer=4, d_model=64, n_head=2, vocab=512, seq_len=64)
LLAMA = E.ModelConfig("tiny-llama", "llama", n_layer=4, d_model=64, n_head=2, vocab=512,
                      seq_len=64, d_ff=176)
GB = 8


def _setup(nodes, groups, n_mb, counts, strategy, cfg=None):
    cfg = cfg or CFG
    prof = E.profile_from_json(E.profile_json(nodes))
    rt = P.fit_runtime_model(prof)
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                        workload=P.WorkloadSpec(GB, CFG.seq_len))
    part = P.make_partition(ctx.graph, groups)
    plan = P.build_plan(ctx, prof, part, n_mb, counts, P.Strategy(strategy),
                        P.cluster_fingerprint(prof), "transformer")
    P.attach_routing(plan, rt, "transformer")
    return plan, ctx


def _run_rank(trainer, steps):
    """Per step, this rank's record for oracle/parity.check_step."""
    ex = trainer.exec
    ex.capture_grads = True
    cfg = ex.cfg
    out = []
    for s in range(1, steps + 1):
        before = parity.snapshot(ex)
        loss = trainer.step(synthetic_batch(cfg.vocab, cfg.seq_len, GB, s))
        out.append(parity.executor_step_record(ex, loss, before))
    return out


def _check(results, steps, cfg=None):
    """Assemble every unit from the ranks' shards (they must tile it exactly once)
    and compare tensor by tensor with the oracle (oracle/parity.py tolerances)."""
    cfg = cfg or CFG
    orc = parity.OracleRun(cfg)
    records = []
    for step in range(1, steps + 1):
        b = synthetic_batch(cfg.vocab, cfg.seq_len, GB, step)
        losses, recs = parity.check_step(cfg, orc, b, step, [r[step - 1] for r in results])
        for got, ref in losses:
            assert parity.loss_ok(got, ref, step), (step, got, ref)
        records += recs
    bad = parity.failures(records)
    assert not bad, parity.describe(records)


@pytest.mark.parametrize("n_mb,counts,strategy", [(1, [1], "zorse"), (2, [4], "zorse"),
                                                  (2, [2], "pp-zero3"), (4, [3], "pp-zero2")])
def test_single_rank_matches_oracle(n_mb, counts, strategy):
    plan, ctx = _setup([("n0", ["b200"])], [["n0-0"]], n_mb, counts, strategy)
    tr = ZorseTrainer(plan, ctx, CFG, _ops=cpu_ops)
    _check([_run_rank(tr, 2)], 2)


@pytest.mark.parametrize("recompute", ["full", "selective", "none"])
@pytest.mark.parametrize("cfg", [CFG, LLAMA], ids=["gpt", "llama"])
def test_recompute_policies_match_oracle(recompute, cfg):
    """The three recompute policies (paper: recompute every block internal from the
    layer checkpoint; selective: keep the attention block's outputs; none: keep the
    whole recompute set) give the same step, two ministages x two microbatches."""
    plan, ctx = _setup([("n0", ["b200"])], [["n0-0"]], 2, [2], "zorse", cfg=cfg)
    tr = ZorseTrainer(plan, ctx, cfg, _ops=cpu_ops, recompute=recompute)
    assert tr.exec.recompute == recompute
    _check([_run_rank(tr, 2)], 2, cfg)


@pytest.mark.parametrize("n_mb,counts", [(4, [1]), (8, [2])])
def test_activation_offload_matches_oracle(n_mb, counts):
    """OffloadAct / LoadAct as real host copies with a 2-microbatch device ring for
    the interior checkpoints (ring slots are reused: M > 2, multi-layer ministages)."""
    plan, ctx = _setup([("n0", ["b200"])], [["n0-0"]], n_mb, counts, "zorse")
    tr = ZorseTrainer(plan, ctx, CFG, _ops=cpu_ops, offload_acts=True)
    ex = tr.exec
    assert ex.offload and any(ex.interior.values())
    ring = {id(t) for t in ex.act.values()}
    assert len(ring) < len(ex.act)          # slots are shared across microbatches
    _check([_run_rank(tr, 2)], 2)


@pytest.mark.parametrize("n_mb,counts,strategy", [(2, [2], "zorse"), (2, [4], "pp-zero3")])
def test_single_rank_llama_matches_oracle(n_mb, counts, strategy):
    plan, ctx = _setup([("n0", ["b200"])], [["n0-0"]], n_mb, counts, strategy, cfg=LLAMA)
    tr = ZorseTrainer(plan, ctx, LLAMA, _ops=cpu_ops)
    _check([_run_rank(tr, 2)], 2, LLAMA)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, spec, q, cfg=None, schedule="gpipe"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan, ctx = _setup(*spec, cfg=cfg)
        def comms(groups_ranks):
            world_c = cpu_ops.GlooComm(list(range(world)), rank)
            group = None
            for ranks in groups_ranks:  # every rank must create every subgroup
                c = cpu_ops.GlooGroupComm(ranks, rank)
                if rank in ranks and len(ranks) > 1:
                    group = c
            return world_c, group
        tr = ZorseTrainer(plan, ctx, cfg or CFG, world_rank=rank, world_size=world, _ops=cpu_ops,
                          _comms=comms, schedule=schedule)
        # plain numpy (tensors in a Queue are shared by fd and die with the worker)
        q.put((rank, _run_rank(tr, 2)))
    except Exception as exc:  # surface worker failures to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec", [
    # 2 asymmetric stages: [n1-0] (1 rank) then [n0-0, n0-1] (uneven 3:1 shares)
    ([("n0", ["b200", "b200h"]), ("n1", ["b200"])], [["n0-0", "n0-1"], ["n1-0"]], 2, [1, 1], "zorse"),
    # interleaved ministages: stages alternate groups (4 global stages)
    ([("n0", ["b200", "b200h"]), ("n1", ["b200"])], [["n0-0", "n0-1"], ["n1-0"]], 2, [2, 2], "zorse"),
    # one uneven DP group of 3 (ZeRO-3 per-microbatch gathers)
    ([("n0", ["b200", "b200", "b200h"])], [["n0-0", "n0-1", "n0-2"]], 2, [2], "pp-zero3"),
], ids=["2stage", "interleaved", "dp3-zero3"])
def test_three_ranks_gloo_matches_oracle(spec):
    _run_gloo(spec, 3)


def _run_gloo(spec, world, cfg=None, schedule="gpipe"):
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _free_port()
    procs = [ctx_mp.Process(target=_worker, args=(r, world, port, spec, q, cfg, schedule))
             for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, res = q.get(timeout=300)
        results[rank] = res
    for p in procs:
        p.join(timeout=60)
    errs = [r for r in results.values() if isinstance(r, str)]
    assert not errs, errs[0]
    _check(list(results.values()), 2, cfg)


@pytest.mark.parametrize("spec,schedule", [
    (([("n0", ["b200", "b200h"]), ("n1", ["b200"])], [["n0-0", "n0-1"], ["n1-0"]], 2, [2, 2],
      "zorse"), "gpipe"),
    (([("n0", ["b200", "b200", "b200h"])], [["n0-0", "n0-1", "n0-2"]], 2, [1], "pp-zero3"),
     "1f1b"),
], ids=["interleaved", "dp3-1f1b"])
def test_windows_gloo(spec, schedule):
    """Parameter / gradient window slots reused across ministages (interleaved
    stages alternating groups) and the PP_ZERO3 two-layer window under 1F1B,
    against the oracle, with a gloo twin of the peer communicator."""
    _run_gloo(spec, 3, CFG, schedule)


def test_1f1b_three_stages_llama_gloo():
    """BASELINE config 4 shape in miniature: Llama, 1F1B, 3 pipeline stages."""
    spec = ([("n0", ["b200"]), ("n1", ["b200"]), ("n2", ["b200h"])],
            [["n0-0"], ["n1-0"], ["n2-0"]], 4, [1, 1, 1], "pp-zero3")
    _run_gloo(spec, 3, LLAMA, "1f1b")


def test_1f1b_two_stages_with_dp_gloo():
    spec = ([("n0", ["b200", "b200h"]), ("n1", ["b200"])], [["n0-0", "n0-1"], ["n1-0"]], 4,
            [1, 1], "pp-zero3")
    _run_gloo(spec, 3, CFG, "1f1b")


def test_1f1b_schedule_shape():
    plan, ctx = _setup([("n0", ["b200"]), ("n1", ["b200"]), ("n2", ["b200"])],
                       [["n0-0"], ["n1-0"], ["n2-0"]], 4, [1, 1, 1], "pp-zero3")
    sched = P.build_schedule(ctx, plan, "1f1b")
    for gi in range(3):
        comp = [(e.kind[0], e.microbatch) for e in sched.stream_for(plan.groups[gi].device_ids[0])
                if e.kind in ("Fwd", "Bwd") and e.group == gi]
        s = plan.global_order().index((gi, 0))
        warm = min(3 - s - 1, 4)
        assert [c for c in comp[:warm]] == [("F", m) for m in range(warm)]
        assert comp[warm:warm + 2] == [("F", warm), ("B", 0)] or warm == 4
        counts = sched.collective_counts()[gi]
        assert counts == {"allgather": 2 * plan.groups[gi].layers_assigned * 4,
                          "reduce_scatter": plan.groups[gi].layers_assigned}


def _faulty(name, wrap):
    """A copy of the CPU twin with one op wrapped (mutation test of the checker)."""
    import types
    m = types.ModuleType("cpu_ops_faulty")
    m.__dict__.update(cpu_ops.__dict__)
    setattr(m, name, wrap(getattr(cpu_ops, name)))
    return m


def _ln_weight_grad_scaled(f):   # LayerNorm dw 3% low: hid inside a unit's norm before
    def g(dy, x, w, mean, rstd, dx, dw, db, *a, **kw):
        before = dw.clone()
        f(dy, x, w, mean, rstd, dx, dw, db, *a, **kw)
        dw.copy_(before + 0.97 * (dw - before))
    return g


def _bias_grad_dropped(f):       # fc1 / qkv bias gradient lost
    return lambda dy, db: None


def _adam_no_bias_correction(f):  # bias-corrected first moment replaced by the raw one
    def g(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, lr, b1, b2, eps, wd, scale, step):
        f(master, exp_avg, exp_avg_sq, grad, param_bf16, sumsq, lr * (1 - b1), b1, b2, eps,
          wd / (1 - b1), scale, step)
    return g


@pytest.mark.parametrize("name,wrap", [("layernorm_bwd", _ln_weight_grad_scaled),
                                       ("bias_grad", _bias_grad_dropped),
                                       ("adamw_shard", _adam_no_bias_correction)],
                         ids=["ln-dw-3pct", "bias-grad-dropped", "adam-bias-correction"])
def test_parity_checker_catches_faults(name, wrap):
    """The per-tensor checks (oracle/parity.py) reject faults that the round-1 per-unit
    gradient bound let through: a 3% error in LayerNorm weight gradients, a dropped
    bias gradient, a wrong Adam step size."""
    plan, ctx = _setup([("n0", ["b200"])], [["n0-0"]], 1, [1], "zorse")
    tr = ZorseTrainer(plan, ctx, CFG, _ops=_faulty(name, wrap))
    with pytest.raises(AssertionError):
        _check([_run_rank(tr, 2)], 2)
