#!/bin/bash
mkdir -p gpurun_out
python scripts/bench_attn.py > gpurun_out/attn_bench.jsonl 2>&1
python scripts/attn_one.py && \
ncu --set full --import-source on --clock-control none -k regex:dkdvq -c 1 -o gpurun_out/attn_bwd_full python scripts/attn_one.py > gpurun_out/attn_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/attn_ncu.log
cat gpurun_out/attn_bench.jsonl; tail -2 gpurun_out/attn_ncu.log
