"""TEST INFRASTRUCTURE ONLY — per-tensor parity of a training step against the
fp32 oracle (SURVEY §8c tolerances).  Used by tests/, scripts/mgpu_check.py and
__graft_entry__.smoke(); never by the product.

A flat parameter unit (a layer, the embedding or the head) is compared tensor by
tensor (``gpt_cpu.unit_entries``), so a small tensor (a LayerNorm weight, a bias)
cannot hide inside a large unit's norm:

* gradient (the reduced, scaled gradient the optimizer consumed):
  rel-L2 <= GRAD_REL and cosine >= GRAD_COS per tensor;
* update delta = p_after - p_before of the fp32 master parameters, two ways:
  (a) optimizer exactness: |delta - AdamW(state, g)| <= OPT_ABS * lr for EVERY
      element, AdamW applied by the oracle rule to the product's own state and
      reduced gradient (pins the fused optimizer arithmetic independently of the
      gradient noise);
  (b) agreement with the oracle's update: at least UPD_FRAC of the elements within
      UPD_ABS * lr of the oracle's delta, over the elements where the update is
      determined by the gradient rather than by bf16 noise: |g_ref| >
      max(NOISE_FLOOR * rms(g_ref), NOISE_SIGMAS * sigma) and AdamW's sensitivity
      d(delta)/dg = lr * (1 - beta1) / ((1 - beta1^t) * sqrt(v_hat_ref)) times
      COND_SIGMAS * sigma stays within UPD_ABS * lr, sigma = rms(g - g_ref) of the
      tensor, the measured gradient noise (itself bounded by the rel-L2 check).
      Adam normalises each element's step (step 1 moves every element by
      ~lr * sign(g)), so the update is compared instead of the parameters;
* first Adam moment exp_avg: rel-L2 <= MOM_REL per tensor;
* loss: relative error <= LOSS_REL_STEP1 at step 1 (identical parameters),
  <= LOSS_REL afterwards.

The bf16 storage / fp32 accumulation of the B200 path is what the tolerances
absorb; every number is written here and in DESIGN.md §3.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional

import torch

from .gpt_cpu import spans, unit_entries

GRAD_REL = 2e-2
GRAD_COS = 0.999
UPD_FRAC = 0.99
UPD_ABS = 0.05        # x lr
NOISE_FLOOR = 0.05    # x rms(g_ref) of the tensor
NOISE_SIGMAS = 10.0   # x rms(g - g_ref) of the tensor
COND_SIGMAS = 4.0
OPT_ABS = 1e-3        # x lr
MOM_REL = 2e-2
LOSS_REL_STEP1 = 2e-3
LOSS_REL = 1e-2


def rel_l2(a: torch.Tensor, b: torch.Tensor) -> float:
    a, b = a.double().flatten(), b.double().flatten()
    return ((a - b).norm() / (b.norm() + 1e-30)).item()


def cosine(a: torch.Tensor, b: torch.Tensor) -> float:
    a, b = a.double().flatten(), b.double().flatten()
    na, nb = a.norm().item(), b.norm().item()
    if na == 0.0 and nb == 0.0:
        return 1.0
    return (a @ b).item() / (na * nb + 1e-300)


def update_agreement(delta: torch.Tensor, ref_delta: torch.Tensor, grad: torch.Tensor,
                     ref_grad: torch.Tensor, ref_v: torch.Tensor, lr: float, step: int,
                     beta1: float = 0.9, beta2: float = 0.95) -> float:
    """Fraction of the gradient-determined elements whose update is within
    UPD_ABS*lr of the oracle's (module docstring, (b))."""
    g = ref_grad.double().flatten()
    if not g.numel():
        return 1.0
    rms = math.sqrt((g * g).mean().item())
    sigma = math.sqrt(((grad.double().flatten() - g) ** 2).mean().item())
    v_hat = ref_v.double().flatten() / (1 - beta2 ** step)
    sens = lr * (1 - beta1) / (1 - beta1 ** step) / (v_hat.sqrt() + 1e-30)
    mask = (g.abs() > max(NOISE_FLOOR * rms, NOISE_SIGMAS * sigma)) & \
        (sens * COND_SIGMAS * sigma <= UPD_ABS * lr)
    if not bool(mask.any()):
        return 1.0
    err = (delta.double().flatten() - ref_delta.double().flatten()).abs()[mask]
    return (err <= UPD_ABS * lr).double().mean().item()


def adamw_expected(p0, m0, v0, g, step, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, wd=0.1):
    """Update the oracle's AdamW rule gives for this state and gradient (fp64)."""
    p0, m0, v0, g = (t.double() for t in (p0, m0, v0, g))
    m = beta1 * m0 + (1 - beta1) * g
    v = beta2 * v0 + (1 - beta2) * g * g
    p = p0 * (1 - lr * wd)
    p = p - lr / (1 - beta1 ** step) * m / ((v / (1 - beta2 ** step)).sqrt() + eps)
    return p - p0


def check_unit(cfg, unit, grad: torch.Tensor, ref_grad: torch.Tensor, *, lr: float,
               step: int = 1, delta: Optional[torch.Tensor] = None,
               ref_delta: Optional[torch.Tensor] = None, ref_v: Optional[torch.Tensor] = None,
               before: Optional[tuple] = None, exp_avg: Optional[torch.Tensor] = None,
               ref_exp_avg: Optional[torch.Tensor] = None, lo: int = 0,
               hi: Optional[int] = None) -> List[dict]:
    """Per-tensor records for the flat range [lo, hi) of ``unit`` (full unit by
    default).  ``grad``, ``delta``, ``exp_avg`` and ``before`` = the product's
    (master, exp_avg, exp_avg_sq) before the step hold that range; ``ref_*`` (the
    oracle's gradient, update, exp_avg and exp_avg_sq after the step) the whole unit."""
    hi = ref_grad.numel() if hi is None else hi
    out = []
    for name, a, b, _shape in spans(unit_entries(cfg, unit)):
        s, e = max(a, lo), min(b, hi)
        if s >= e:
            continue
        mine = slice(s - lo, e - lo)
        ref = slice(s, e)
        rec = {"unit": str(unit), "tensor": name, "numel": e - s,
               "grad_rel": rel_l2(grad[mine], ref_grad[ref]),
               "grad_cos": cosine(grad[mine], ref_grad[ref])}
        ok = rec["grad_rel"] <= GRAD_REL and rec["grad_cos"] >= GRAD_COS
        if delta is not None:
            rec["upd_frac"] = update_agreement(delta[mine], ref_delta[ref], grad[mine],
                                               ref_grad[ref], ref_v[ref], lr, step)
            ok = ok and rec["upd_frac"] >= UPD_FRAC
        if before is not None:
            exp = adamw_expected(*(t[mine] for t in before), grad[mine], step, lr=lr)
            rec["opt_err"] = (delta[mine].double() - exp).abs().max().item() / lr
            ok = ok and rec["opt_err"] <= OPT_ABS
        if exp_avg is not None:
            rec["mom_rel"] = rel_l2(exp_avg[mine], ref_exp_avg[ref])
            ok = ok and rec["mom_rel"] <= MOM_REL
        rec["ok"] = ok
        out.append(rec)
    return out


def loss_ok(loss: float, ref_loss: float, step: int) -> bool:
    tol = LOSS_REL_STEP1 if step == 1 else LOSS_REL
    return abs(loss - ref_loss) / abs(ref_loss) <= tol


def failures(records: List[dict]) -> List[dict]:
    return [r for r in records if not r["ok"]]


def worst(records: List[dict]) -> Dict[str, object]:
    """Summary: worst value of each metric with the tensor it came from."""
    out: Dict[str, object] = {"tensors": len(records), "failed": len(failures(records))}
    for key, pick in (("grad_rel", max), ("grad_cos", min), ("upd_frac", min), ("mom_rel", max),
                      ("opt_err", max)):
        vals = [(r[key], f"{r['unit']}.{r['tensor']}") for r in records if key in r]
        if vals:
            v, where = pick(vals, key=lambda t: t[0])
            out[key] = v
            out[key + "_at"] = where
    return out


def describe(records: List[dict], limit: int = 6) -> str:
    """One-line summary plus the first failing records (assertion messages)."""
    import json
    bad = failures(records)
    return json.dumps({"worst": worst(records), "failures": bad[:limit]}, default=str)


class OracleRun:
    """The oracle's side of a multi-step comparison (gpt_cpu.adamw rule).

    Each step is compared from the SAME state: ``step(batch, sync)`` first loads the
    product's fp32 master parameters and Adam moments as they were before that step
    (``sync = {unit: (master, exp_avg, exp_avg_sq)}``, full units).  Without it, step
    t > 1 would compare gradients taken at different parameters — Adam's step-1
    update is ~lr*sign(g), so an element whose gradient is below the bf16 noise
    flips by 2*lr and the trajectories separate (chaotically) from there."""

    def __init__(self, cfg, seed: int = 1234, **adam_kw):
        from . import gpt_cpu
        self.cfg = cfg
        self.params = gpt_cpu.init_params(cfg, seed)
        self.state: dict = {}
        self.adam_kw = adam_kw
        self.step_no = 0

    def step(self, batch, sync=None):
        """Returns (loss, grads, deltas, exp_avgs, exp_avg_sqs) of this step."""
        from . import gpt_cpu
        self.step_no += 1
        if sync is not None:
            for k, (p, m, v) in sync.items():
                self.params[k] = p.detach().float().cpu().clone()
                self.state[k] = (m.detach().float().cpu().clone(), v.detach().float().cpu().clone())
        before = {k: v.clone() for k, v in self.params.items()}
        loss, grads = gpt_cpu.loss_and_grads(self.cfg, self.params, batch)
        gpt_cpu.adamw(self.params, grads, self.state, self.step_no, **self.adam_kw)
        deltas = {k: self.params[k] - before[k] for k in self.params}
        moms = {k: self.state[k][0].clone() for k in self.params}
        sq = {k: self.state[k][1].clone() for k in self.params}
        return loss, grads, deltas, moms, sq


def check_step(cfg, orc: "OracleRun", batch, step: int, rank_steps: List[dict],
               lr: float = 1e-3) -> tuple:
    """Assemble one step's per-rank shard records into full units and compare with
    the oracle step taken from the same (synced) state.

    rank_steps: one dict per rank {"loss": float, "shards": {unit: (lo, hi, grad,
    delta, exp_avg, master0, exp_avg0, exp_avg_sq0)}} (numpy or torch arrays; the
    last three = state before the step).  Shards of a unit must tile it exactly
    once.  Returns (loss pairs [(rank loss, oracle loss)], records)."""
    import numpy as np
    full: Dict[object, list] = {}
    for r in rank_steps:
        for u, shard in r["shards"].items():
            full.setdefault(u, []).append(shard)
    cat = {}
    for u, parts in full.items():
        parts.sort(key=lambda t: t[0])
        if parts[0][0] != 0 or any(a[1] != b[0] for a, b in zip(parts, parts[1:])):
            raise AssertionError(f"shards of unit {u} do not tile it: "
                                 f"{[(p[0], p[1]) for p in parts]}")
        cat[u] = [torch.as_tensor(np.concatenate([np.asarray(p[k]) for p in parts]))
                  for k in range(2, 8)]
    ref_loss, ref_g, ref_d, ref_m, ref_v = orc.step(batch, sync={u: c[3:] for u, c in cat.items()})
    records = []
    for u, c in cat.items():
        if c[0].numel() != ref_g[u].numel():
            raise AssertionError(f"unit {u}: shards cover {c[0].numel()} of {ref_g[u].numel()}")
        recs = check_unit(cfg, u, c[0], ref_g[u], lr=lr, step=step, delta=c[1],
                          ref_delta=ref_d[u], ref_v=ref_v[u], before=c[3:], exp_avg=c[2],
                          ref_exp_avg=ref_m[u])
        for rec in recs:
            rec["step"] = step
        records += recs
    return [(r["loss"], ref_loss) for r in rank_steps], records


def executor_step_record(ex, loss: float, before: dict) -> dict:
    """One rank's record for check_step from a StageExecutor after a step run with
    ``capture_grads``; ``before`` = {unit: (master, exp_avg, exp_avg_sq)} clones taken
    before the step.  Arrays are numpy (they cross process boundaries)."""
    sh = {}
    for u, pu in ex.units.items():
        p0, m0, v0 = before[u]
        arrs = (ex.captured[u].float(), pu.master - p0, pu.exp_avg, p0, m0, v0)
        sh[u] = (pu.lo, pu.hi, *[t.detach().cpu().clone().numpy() for t in arrs])
    return {"loss": loss, "shards": sh}


def snapshot(ex) -> dict:
    return {u: (pu.master.detach().clone(), pu.exp_avg.detach().clone(),
                pu.exp_avg_sq.detach().clone()) for u, pu in ex.units.items()}
