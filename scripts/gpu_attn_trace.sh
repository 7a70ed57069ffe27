#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/attn_trace.py paper_2507_10392_b200/libzorse_trace.so > gpurun_out/attn_trace.log 2>&1
echo rc=$?
tail -n 12 gpurun_out/attn_trace.log
