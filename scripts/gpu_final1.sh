#!/bin/bash
# Single-GPU round-end evidence: tests, smoke, bench (ours + reference arm),
# ncu launch list of the bench command, GEMM DRAM traffic, one full ncu capture.
O=gpurun_out/final1
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/summary.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 3 --warmup 3 --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/summary.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemm --csv --log-file $O/gemm_dram.csv python scripts/profile_step.py 1 > $O/ncu_dram.log 2>&1; echo "ncu dram rc=$?" >> $O/summary.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 20 -c 2 \
  -o $O/gemm_step_full python scripts/profile_step.py 1 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/summary.log
