#!/bin/bash
# compute-sanitizer over one call of every kernel family (scripts/sanitize_kernels.py).
mkdir -p gpurun_out
python scripts/sanitize_kernels.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_kernels.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -n 4 gpurun_out/sanitize_*.log
