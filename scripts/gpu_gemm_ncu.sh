#!/bin/bash
# GEMM evidence of the current step: DRAM bytes of every GEMM launch of one eager step
# (bench roofline `traffic`), a full ncu capture of three step GEMMs, and the launch list.
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --eager > gpurun_out/plain_eager.json 2>/dev/null && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:gemm -c 147 --csv --log-file gpurun_out/gemm_dram_r02.csv python bench.py --steps 1 --warmup 1 --eager > /dev/null 2>&1; echo "dram rc=$?"
ncu --set full --import-source on --clock-control none -k regex:gemm --launch-skip 4 -c 3 \
    -o gpurun_out/gemm_step_full_r02 python bench.py --steps 1 --warmup 1 --eager > /dev/null 2>&1; echo "full rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 > /dev/null 2>&1; echo "ll rc=$?"
python scripts/gemm_traffic.py gpurun_out/gemm_dram_r02.csv gpurun_out/gemm_traffic.json
python scripts/launch_summary.py gpurun_out/launches_r02.csv 4 | head -32
