"""Benchmark: device-timed training tokens/s of the Zorse hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by the driver with torchrun (one process per GPU).  The
workload is BASELINE config 2 — GPT-2 small (124M), seq 1024, one pipeline
stage x an N-rank uneven ZeRO-3 DP group whose per-device batch shares come
from the planner on an emulated-heterogeneity profile (half b200, half
half-speed b200h), 8 sequences per GPU on average (weak scaling; at N=8 this
is exactly config 2: global batch 64, shares 11x4 / 5x4).

ours      : the B200 executor (tcgen05 GEMMs and flash attention, AG-v and fused
            RS-v + AdamW over NVLink peer memory) — value = whole-job tokens/s, device-timed,
            max over ranks; e2e = same metric through ZorseTrainer.step with
            the batch in pinned host memory and the loss read back each step.
reference : the reference has no training step (hetplan is a planner +
            simulator); its CPU path for this metric is the oracle port
            (oracle/gpt_cpu.py, fp32 torch on all host cores): K timed + W warm-up
            full training steps of 8 x 1024 tokens (the whole N=1 step; a bounded
            sample of the 8N-sequence batch at N>1), rank 0 only, no product code
            in the process.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return p, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


def build_workload(n_gpus: int, per_gpu_batch: int = 8, cfg=None):
    """GPT-2 small (or ``cfg``: tile tuning of other models' shapes), one stage x an
    n_gpus-rank uneven ZeRO-3 DP group (product planner)."""
    from paper_2507_10392_b200 import plan as P
    from paper_2507_10392_b200.plan import emulated as E

    cfg = cfg or E.GPT2_SMALL
    prof = E.profile_from_json(E.profile_json(E.dp_group_nodes(n_gpus)))
    rt = P.fit_runtime_model(prof)
    gb = per_gpu_batch * n_gpus
    ctx = P.CostContext(graph=P.build_cluster_graph(prof), runtime=rt, model=cfg.model_spec(),
                        workload=P.WorkloadSpec(gb, cfg.seq_len))
    part = P.make_partition(ctx.graph, [[d.id for d in prof.devices]])
    plan = P.build_plan(ctx, prof, part, 1, [cfg.n_layer], P.Strategy.INTERLEAVED,
                        P.cluster_fingerprint(prof), "transformer")
    P.attach_routing(plan, rt, "transformer")
    return cfg, plan, ctx, gb


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class TimedOps:
    """Wraps the kernel module: CUDA events around every GEMM launch (same stream)."""

    def __init__(self, ops):
        self.ops = ops
        self.records = []
        self.bytes = []

    def __getattr__(self, name):
        return getattr(self.ops, name)

    def gemm(self, a, b, out, **kw):
        a_t, b_t = kw.get("a_t", False), kw.get("b_t", False)
        M = a.shape[1] if a_t else a.shape[0]
        K = a.shape[0] if a_t else a.shape[1]
        N = b.shape[1] if b_t else b.shape[0]
        kw_ev = {"external": True} if getattr(self, "external", False) else {}
        s = torch.cuda.Event(enable_timing=True, **kw_ev)
        e = torch.cuda.Event(enable_timing=True, **kw_ev)
        s.record()
        r = self.ops.gemm(a, b, out, **kw)
        e.record()
        self.records.append((s, e, 2.0 * M * N * K))
        # algorithmic DRAM bytes: A and B read once, C written once (+ read for beta)
        c_bytes = M * N * out.element_size() * (2 if kw.get("beta", 0.0) else 1)
        self.bytes.append(2.0 * (M * K + N * K) + c_bytes)
        return r


PER_GPU_BATCH = 8


def oracle_steps(steps: int, warmup: int, n_seq: int):
    """The CPU path of this metric: oracle/gpt_cpu.py (fp32 torch on every host core;
    the reference itself has no training step) doing full training steps — forward,
    backward and AdamW over all 124M parameters — on batches of ``n_seq`` x 1024
    synthetic tokens of the bench workload.  Imports nothing from the product (its
    CUDA library stays out of this process).  Returns (tokens/s, seconds per timed
    step, threads)."""
    from oracle import gpt_cpu

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    cfg = gpt_cpu.GPT2_SMALL
    params = gpt_cpu.init_params(cfg, 1234)
    state = {}
    for step in range(1, warmup + 1):
        _, grads = gpt_cpu.loss_and_grads(cfg, params, gpt_cpu.synthetic_batch(cfg, n_seq, step))
        gpt_cpu.adamw(params, grads, state, step)
    t0 = time.perf_counter()
    for step in range(warmup + 1, warmup + steps + 1):
        _, grads = gpt_cpu.loss_and_grads(cfg, params, gpt_cpu.synthetic_batch(cfg, n_seq, step))
        gpt_cpu.adamw(params, grads, state, step)
    el = time.perf_counter() - t0
    return steps * n_seq * cfg.seq_len / el, el / steps, threads


L2_POLICY = "per-step working set (params+grads+activations) >> 126 MB L2; no flush"


def workload_config(n: int) -> dict:
    """The `config` object both arms print (identical dicts, so the driver can
    compare them); run-specific details go in the line's `details`."""
    return {"workload": f"gpt2-small-124m (L12 d768 s1024) 1 stage x {n}-rank "
                        "uneven ZeRO-3 DP, planner shares",
            "model": "gpt2-small-124m", "global_batch": PER_GPU_BATCH * n, "seq_len": 1024,
            "parallelism": f"dp{n}", "l2": L2_POLICY}


def cpu_baseline_sample():
    """Bounded CPU sample for the GPU arm's cpu_baseline (rank 0, N=1): one warm-up
    and one timed oracle step of the full N=1 workload (8 x 1024 tokens)."""
    v, s_per, threads = oracle_steps(1, 1, PER_GPU_BATCH)
    return {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"1 timed (+1 warm-up) oracle training step of {PER_GPU_BATCH} x 1024 tokens "
                      f"(GPT-2 small fp32 fwd+bwd+AdamW, oracle/gpt_cpu.py) on {threads} host "
                      f"threads, {s_per:.1f} s/step"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    gb = PER_GPU_BATCH * args.gpus
    # N=1: every step is the full workload step (8 x 1024 tokens).  N>1: the global
    # batch is 8N sequences; each CPU step is a bounded sample of 8 of them (the
    # tokens/s rate of a full step, which would take N times longer).
    v, s_per, threads = oracle_steps(args.steps, args.warmup, PER_GPU_BATCH)
    sample = (f"{args.steps} timed + {args.warmup} warm-up oracle training steps, each "
              f"{PER_GPU_BATCH} x 1024 tokens (" +
              ("the full N=1 step" if args.gpus == 1 else
               f"a bounded sample of the {gb}-sequence global batch") +
              f"), GPT-2 small fp32 fwd+bwd+AdamW (oracle/gpt_cpu.py), {threads} host threads")
    line = {
        "impl": "reference", "metric": "training tokens/sec (device-timed)", "value": v,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": s_per * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (uniform tokens, random init)",
        "config": workload_config(args.gpus),
        "tokens_per_timed_step": PER_GPU_BATCH * 1024,
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


NVLINK_PEER_GBS = 770.0   # measured B200 peer copy per direction (B200_PROFILING.md)


def measure_collectives(trainer, dist, iters=20):
    """AG-v and fused RS-v+AdamW GB/s on the largest parameter unit of this rank's
    group, through the executor's own communicator (the NVLink peer path), after
    the timed region.  AG re-gathers identical values; RS+AdamW writes scratch
    optimizer state, so the trained state is untouched.  Time = max over ranks;
    bytes = what the slowest rank moves over NVLink."""
    import types
    ex = trainer.exec
    comm = ex.group_comm
    if comm is None:
        return None
    key = max(ex.units, key=lambda k: ex.units[k].numel)
    pu = ex.units[key]
    g = len(pu.counts)
    P = pu.numel
    shard = pu.hi - pu.lo
    stage = next(s for s, units in ex.chunks.items() if key in units)
    goff = ex.grad_lo + ex.win.grad_slot[stage] * ex.grad_slot_bytes + ex._grad_unit_off[key]
    full = torch.empty(P, device=pu.master.device, dtype=torch.bfloat16)   # window slot stand-in
    scratch = types.SimpleNamespace(   # the unit's gradient slot (same offset on every rank)
        grad_off=goff, flag_off=pu.flag_off, lo=pu.lo, hi=pu.hi,
        grad=ex.arena.view(goff, P, torch.float32), master=pu.master.clone(),
        exp_avg=pu.exp_avg.clone(), exp_avg_sq=pu.exp_avg_sq.clone(),
        shard=torch.empty_like(pu.shard))
    sumsq = torch.zeros(1, device=pu.master.device)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def maxed(x):
        t = torch.tensor([float(x)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    ag_ms = timeit(lambda: comm.gather(pu, full, ex.step_dev))
    rs_ms = timeit(lambda: comm.reduce_scatter_adamw(scratch, ex.adam, sumsq, ex.step_dev))
    ag_bytes = maxed((P - shard) * 2)                 # bf16 received from peers
    rs_bytes = maxed((g - 1) * shard * 4)             # fp32 peer slices read
    out = {"unit": str(key), "params": P, "group_size": g, "peak_gbs": NVLINK_PEER_GBS,
           "peak_source": "measured peer copy, B200_PROFILING.md"}
    for name, ms, b, how in (("allgather_v", ag_ms, ag_bytes, "copy engines over NVLink peer memory"),
                             ("reduce_scatter_v+adamw", rs_ms, rs_bytes,
                              "one kernel: NVLink loads + sum + AdamW + bf16 cast")):
        gbs = b / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "nvlink_bytes": int(b), "gbs": gbs,
                     "frac": gbs / NVLINK_PEER_GBS, "path": how}
    return out


def run_ours(args):
    from paper_2507_10392_b200 import kernels
    from paper_2507_10392_b200.runtime.data import synthetic_batch
    from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, plan, ctx, gb = build_workload(args.gpus)
    trainer = ZorseTrainer(plan, ctx, cfg, world_rank=rank, world_size=world)
    ex = trainer.exec
    batch = synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True)
    h2d = trainer.load(batch)
    tokens_per_step = gb * cfg.seq_len

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(max(1, args.warmup - 1)):
        trainer.run()                 # eager warm-up (JIT-free: warms TMA maps, NCCL, allocs)
    if not args.eager:
        trainer.capture()             # whole step -> one CUDA graph
    trainer.run()
    torch.cuda.synchronize()
    barrier()

    # ---------------- device-timed region (inputs resident in HBM) ----------------
    kernels.reset_launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        start.record()
        for _ in range(args.steps):
            trainer.run()
        end.record()
        torch.cuda.synchronize()
        barrier()
    launches = kernels.launch_count()
    if trainer.graph is not None:   # replays bypass the Python launch counter
        launches = trainer.launches_per_step * args.steps
    ms = start.elapsed_time(end)
    t = torch.tensor([ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    loss = trainer.loss_device().item()

    # ---------------- e2e through the public API (pinned host batch, loss D2H) ----
    # as many steps as the device-timed region, so both see the same clock / power state
    e2e_steps = max(2, args.steps)
    barrier()
    torch.cuda.synchronize()
    e0 = time.perf_counter()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record()
    for i in range(e2e_steps):
        trainer.step(batch)          # H2D of this rank's tokens/labels + step + loss D2H
    ee.record()
    torch.cuda.synchronize()
    e2e_ms = es.elapsed_time(ee)
    t = torch.tensor([e2e_ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = t.item()

    coll = measure_collectives(trainer, dist) if world > 1 else None

    # ---------------- roofline of the dominant kernel (tcgen05 GEMM) ------------
    timed = TimedOps(kernels)
    ex.ops = timed
    ex.model.ops = timed
    # Per-launch durations are taken with the weight-gradient lane serialised: kernels
    # running concurrently share the SMs, so their event-bracketed times would each
    # include the other's work.  The share of the step is against this serial step.
    wlane = getattr(ex.model, "wlane", None)
    lane_on = bool(wlane and wlane.enabled)
    if wlane is not None:
        wlane.enabled = False
    torch.cuda.synchronize()
    serial_ms = None
    try:  # time GEMMs inside a replayed graph of the step (no host gaps)
        timed.external = True
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            ex.step()
        g2.replay()  # warm-up replay; the second one below re-records the same events
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        g2.replay()
        e2.record()
        torch.cuda.synchronize()
        serial_ms = s2.elapsed_time(e2)
        mode = "graph"
    except Exception:
        timed.records.clear()
        timed.external = False
        ex.step()
        mode = "eager"
    torch.cuda.synchronize()
    if wlane is not None:
        wlane.enabled = lane_on
    ex.ops = kernels
    ex.model.ops = kernels
    g_ms = sum(s.elapsed_time(e) for s, e, _ in timed.records)
    g_flops = sum(f for _, _, f in timed.records)
    n_launch = len(timed.records)
    peaks, src = _peaks()
    peak = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")))
    achieved = g_flops / (g_ms * 1e-3) / 1e12 if g_ms > 0 else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")

    if rank == 0:
        step_flops = cfg.flops_per_token() * tokens_per_step
        line = {
            "metric": "training tokens/sec (device-timed)",
            "value": tokens_per_step * args.steps / (ms * 1e-3),
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (uniform tokens, random init)",
            "config": workload_config(world),
            "details": {
                "shares": [plan.groups[0].shares[d] for d in plan.groups[0].device_ids],
                "n_microbatches": plan.n_microbatches, "ministages": len(plan.groups[0].ministage_sizes),
                "collectives": "nvlink peer memory" if world > 1 else None,
                "recompute": ex.recompute,
                "max_memory_allocated_gib": torch.cuda.max_memory_allocated() / 2**30,
            },
            "loss": loss,
            "model_tflops_per_gpu": step_flops * args.steps / (ms * 1e-3) / 1e12 / world,
            "mfu_of_measured_sustained": step_flops * args.steps / (ms * 1e-3) / 1e12 / world / peak,
            "e2e": {"value": tokens_per_step * e2e_steps / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": 4 * world},
            "gpu_launches": launches,
            "roofline": {"bound": "tensor", "kernel": "zb_gemm_bf16 (tcgen05)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "peak_source": f"{src} bf16_tflops_sustained",
                         "gemm_share_of_step": g_ms / (serial_ms or ms / args.steps),
                         "share_basis": "serial step (weight-gradient lane off)"
                         if serial_ms else "timed step",
                         "launches_per_step": n_launch, "timing_mode": mode,
                         "algorithmic_flops_per_step": g_flops,
                         "algorithmic_bytes_per_launch": (sum(timed.bytes) / len(timed.bytes)
                                                          if timed.bytes else None),
                         "traffic_source": "profiles/gemm_traffic.json (ncu dram bytes, cold "
                                           "cache, every GEMM launch of one step)"},
            "clocks": clocks.summary(),
        }
        if coll is not None:
            line["collectives"] = coll
        if world == 1:
            line["cpu_baseline"] = cpu_baseline_sample()
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--eager", action="store_true", help="no CUDA-graph capture of the step")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
