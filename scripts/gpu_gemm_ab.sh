#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
python scripts/gemm_ab.py paper_2507_10392_b200/libzorse_b200_old.so > gpurun_out/gemm_ab_old_$i.jsonl 2>&1
python scripts/gemm_ab.py > gpurun_out/gemm_ab_new_$i.jsonl 2>&1
done
python - <<'PY'
import json
def load(f): return {d["gemm"]: d for d in map(json.loads, open(f)) }
for i in (1, 2):
    o, n = load(f"gpurun_out/gemm_ab_old_{i}.jsonl"), load(f"gpurun_out/gemm_ab_new_{i}.jsonl")
    for k in o: print(i, f"{k:28s} old {o[k]['tflops']:7.1f} new {n[k]['tflops']:7.1f} TF/s  x{n[k]['tflops']/o[k]['tflops']:.3f} {n[k]['tile']}")
PY
