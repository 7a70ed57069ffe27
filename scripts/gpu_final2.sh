#!/bin/bash
# Tune-cache population (bench N=1 shapes + step shapes), then ncu evidence without
# tuning launches.
O=gpurun_out/final2
mkdir -p $O
rm -f paper_2507_10392_b200/gemm_tune_cache.txt
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/summary.log
timeout 300 python scripts/profile_step.py 1 > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/summary.log
cp paper_2507_10392_b200/gemm_tune_cache.txt $O/gemm_tune_cache.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/summary.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemm --csv --log-file $O/gemm_dram.csv python scripts/profile_step.py 1 > $O/ncu_dram.log 2>&1; echo "ncu dram rc=$?" >> $O/summary.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 20 -c 2 \
  -o $O/gemm_step_full python scripts/profile_step.py 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/summary.log
timeout 300 python scripts/step_breakdown.py --json $O/breakdown.json > $O/breakdown.txt 2>&1; echo "breakdown rc=$?" >> $O/summary.log
