#!/bin/bash
mkdir -p gpurun_out
python scripts/gemm_ab.py > gpurun_out/gemm_ab_new_1.jsonl 2>&1
cat gpurun_out/gemm_ab_new_1.jsonl | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(f\"{d['gemm']:28s} {d['us']:8.1f} us {d['tflops']:7.1f} TF/s tile {d['tile']}\")"
