"""TEST INFRASTRUCTURE ONLY — CPU oracle for the Zorse B200 hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the CPU
baseline.  The product (paper_2507_10392_b200) never imports it.

* gpt_cpu.py  — fp32 torch-CPU restatement of one training step (forward,
  backward, AdamW) for the GPT model the executor runs.
* The plan / schedule / shard-layout oracle is the REFERENCE itself (hetplan,
  imported in the build container) frozen into tests/golden/ by
  tests/golden/make_golden.py.

Parity of the arithmetic (loss, gradients, updated parameters) is NOT pinned
by the reference: hetplan has no tensor math.  This oracle follows
the semantics the paper states (per-layer checkpointing with
recompute, per-ministage optimizer) — none of which changes the arithmetic of
a step, so the oracle is a plain full-batch fp32 step.
"""
