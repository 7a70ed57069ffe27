#!/bin/bash
# Round evidence: launch list of the bench step, full ncu captures of the attention
# kernels and the cross-entropy (each after its plain run exited 0).
mkdir -p gpurun_out
bash scripts/gpu_launches.sh
python scripts/attn_one.py && \
ncu --set full --import-source on --clock-control none -k regex:"dkdvq|fwd_pp" -c 2 -o gpurun_out/attn_full_r02b python scripts/attn_one.py > gpurun_out/attn_ncu.log 2>&1; echo "attn ncu rc=$?"
python scripts/xent_bench.py && \
ncu --set full --clock-control none -k regex:xent -c 1 -o gpurun_out/xent_full_r02b python scripts/xent_bench.py > gpurun_out/xent_ncu.log 2>&1; echo "xent ncu rc=$?"
for f in attn_full_r02b xent_full_r02b; do
  ncu -i gpurun_out/$f.ncu-rep --page details --csv > gpurun_out/$f.details.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
