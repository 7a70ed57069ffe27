"""End-to-end training steps on one B200 through the product path (C-ABI
kernels), against the CPU fp32 oracle.  Tolerances (bf16 storage, fp32
accumulate): loss rel <= 1e-2; per-unit gradient rel-L2 <= 3e-2; master params
after 2 AdamW steps within 2*2.5e-3 absolute (lr 1e-3 => <= ~1.25 lr per step)."""

import pytest
import torch

from oracle import gpt_cpu
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


def _rel(a, b):
    return ((a - b).norm() / (b.norm() + 1e-12)).item()


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
def test_training_steps_match_oracle(cuda, cfg, gb, n_mb, counts, strategy, offload):
    plan, ctx = _setup(cfg, gb, n_mb, counts, strategy)
    tr = ZorseTrainer(plan, ctx, cfg, offload_acts=offload)
    assert tr.exec.offload == offload
    tr.exec.capture_grads = True
    batches = [synthetic_batch(cfg.vocab, cfg.seq_len, gb, s) for s in (1, 2)]
    params = gpt_cpu.init_params(cfg, 1234)
    state = {}
    for step, b in enumerate(batches, start=1):
        loss = tr.step(b.pin_memory())
        ref_loss, ref_grads = gpt_cpu.loss_and_grads(cfg, params, b)
        gpt_cpu.adamw(params, ref_grads, state, step)
        assert abs(loss - ref_loss) / ref_loss < 1e-2, (step, loss, ref_loss)
        wide = cfg.d_model >= 4096
        for u, g in tr.exec.captured.items():
            r = _rel(g.cpu(), ref_grads[u])
            if wide and step > 1:
                cos = torch.nn.functional.cosine_similarity(g.cpu().flatten(),
                                                            ref_grads[u].flatten(), dim=0).item()
                assert r < 5e-2 and cos >= 0.998, (step, u, r, cos)
            else:
                assert r < 3e-2, (step, u, r)
    for u, pu in tr.exec.units.items():
        err = (pu.master.cpu() - params[u]).abs().max().item()
        assert err < 5e-3, (u, err)
