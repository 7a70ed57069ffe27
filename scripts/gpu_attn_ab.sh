#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k attention -p no:cacheprovider 2>&1 | tail -n 1
for i in 1 2; do
python scripts/bench_attn.py paper_2507_10392_b200/libzorse_b200_old.so > gpurun_out/attn_old.jsonl
python scripts/bench_attn.py > gpurun_out/attn_new.jsonl
python -c "
import json
o=[json.loads(l) for l in open('gpurun_out/attn_old.jsonl')]; n=[json.loads(l) for l in open('gpurun_out/attn_new.jsonl')]
for a,b in zip(o,n): print(a['shape'], 'fwd', round(a['fwd_tflops']), '->', round(b['fwd_tflops']), 'bwd', round(a['bwd_tflops(2.5x fwd flops)']), '->', round(b['bwd_tflops(2.5x fwd flops)']))"
done
