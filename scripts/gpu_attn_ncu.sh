#!/bin/bash
mkdir -p gpurun_out
python scripts/attn_one.py && \
ncu --set full --import-source on --clock-control none -k regex:"dkdvq|fwd_pp" -c 2 -o gpurun_out/attn_full python scripts/attn_one.py > gpurun_out/attn_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/attn_ncu.log; tail -2 gpurun_out/attn_ncu.log
