#!/bin/bash
# Planner-loop reports (4 GPUs) + NVLink probe of the peer collectives with ncu counters.
mkdir -p gpurun_out
bash scripts/gpu_report.sh > gpurun_out/gpu_report.log 2>&1
python scripts/nvlink_probe.py > gpurun_out/nvlink_probe.jsonl 2> gpurun_out/nvlink_probe.err && \
python scripts/nvlink_probe.py --ncu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:peer_ --csv --log-file gpurun_out/nvlink_ncu.csv python scripts/nvlink_probe.py --ncu > gpurun_out/nvlink_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/nvlink_ncu.log
cat gpurun_out/nvlink_probe.jsonl | cut -c1-200; tail -3 gpurun_out/nvlink_ncu.log; tail -20 gpurun_out/gpu_report.log
