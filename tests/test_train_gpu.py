"""End-to-end training steps on one B200 through the product path (C-ABI
kernels), against the CPU fp32 oracle, tensor by tensor (oracle/parity.py):
step-1 loss rel <= 2e-3 (later steps 1e-2); every named tensor's reduced gradient
rel-L2 <= 2e-2 with cosine >= 0.999; >= 99% of the above-noise-floor elements of
every tensor's fp32 master update within 0.05*lr of the oracle's update; exp_avg
rel-L2 <= 2e-2."""

import pytest
import torch

from oracle import parity
from paper_2507_10392_b200 import plan as P
from paper_2507_10392_b200.plan import emulated as E
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

pytestmark = pytest.mark.gpu


def _setup(cfg, gb, n_mb, counts, strategy):
    prof = E.profile_from_json(E.profile_json([("n0", ["b200"])]))
    rt = P.fit_runtime_model(prof)
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                        workload=P.WorkloadSpec(gb, cfg.seq_len))
    plan = P.build_plan(ctx, prof, P.make_partition(ctx.graph, [["n0-0"]]), n_mb, counts,
                        P.Strategy(strategy), P.cluster_fingerprint(prof), "transformer")
    P.attach_routing(plan, rt, "transformer")
    return plan, ctx


def run_and_compare(tr, cfg, batches, lr=1e-3):
    """Steps the trainer and the oracle side by side (oracle synced to the product's
    state before each step); returns (loss triples, per-tensor records)."""
    ex = tr.exec
    ex.capture_grads = True
    orc = parity.OracleRun(cfg)
    losses, records = [], []
    for step, b in enumerate(batches, start=1):
        before = parity.snapshot(ex)
        loss = tr.step(b.pin_memory())
        pairs, recs = parity.check_step(cfg, orc, b, step,
                                        [parity.executor_step_record(ex, loss, before)], lr)
        losses += [(step, got, ref) for got, ref in pairs]
        records += recs
    return losses, records


@pytest.mark.parametrize("cfg,gb,n_mb,counts,strategy,offload", [
    (E.TINY_GPT, 8, 2, [1], "zorse", False),                  # BASELINE config 1 model
    (E.TINY_GPT, 8, 2, [4], "pp-zero3", False),
    (E.ModelConfig("mid", "gpt", 2, 768, 12, 4096, 1024), 2, 1, [2], "zorse", False),  # GPT-2 widths
    (E.ModelConfig("llama-tiny", "llama", 2, 512, 4, 4096, 256, d_ff=1376), 4, 2, [2], "zorse", False),
    (E.ModelConfig("llama-hd128", "llama", 2, 1024, 8, 4096, 512, d_ff=2752), 2, 1, [1], "pp-zero3",
     False),
    # Llama-13B widths (BASELINE config 5): d 5120, 40 heads of 128, d_ff 13824.  bf16
    # activations over K = 13824 drift further from fp32 after one update: the step-2
    # gradient bound is the multi-GPU one (rel-L2 <= 5e-2 with cosine >= 0.998)
    (E.ModelConfig("llama13b-width", "llama", 1, 5120, 40, 2048, 256, d_ff=13824), 2, 1, [1],
     "zorse", False),
    # activation offload to pinned host memory (OffloadAct / LoadAct on the host stream)
    (E.TINY_GPT, 8, 4, [1], "zorse", True),
])
@pytest.mark.parametrize("recompute", ["auto", "full"])
def test_training_steps_match_oracle(cuda, cfg, gb, n_mb, counts, strategy, offload, recompute):
    plan, ctx = _setup(cfg, gb, n_mb, counts, strategy)
    tr = ZorseTrainer(plan, ctx, cfg, offload_acts=offload, recompute=recompute)
    assert tr.exec.offload == offload
    batches = [synthetic_batch(cfg.vocab, cfg.seq_len, gb, s) for s in (1, 2)]
    losses, records = run_and_compare(tr, cfg, batches)
    for step, loss, ref in losses:
        assert parity.loss_ok(loss, ref, step), (step, loss, ref)
    bad = parity.failures(records)
    assert not bad, parity.describe(records)
