#!/bin/bash
# Single-GPU round-end evidence (round 1, second session): tests, smoke, bench (both
# arms), ncu launch list of the bench command, GEMM DRAM traffic, full ncu captures of
# the top kernels, in-step breakdown.
O=gpurun_out/r1b_final1b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/summary.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/summary.log
timeout 600 python bench.py --steps 3 --warmup 3 --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/summary.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/summary.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemm --csv --log-file $O/gemm_dram.csv python scripts/profile_step.py 1 > $O/ncu_dram.log 2>&1; echo "ncu dram rc=$?" >> $O/summary.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm -s 20 -c 3 \
  -o $O/gemm_step_full python scripts/profile_step.py 1 > $O/ncu_full.log 2>&1; echo "ncu full gemm rc=$?" >> $O/summary.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fwd_pp|dkdvq" -s 2 -c 2 \
  -o $O/attn_step_full python scripts/profile_step.py 1 > $O/ncu_attn.log 2>&1; echo "ncu full attn rc=$?" >> $O/summary.log
timeout 300 python scripts/step_breakdown.py --json $O/breakdown.json > $O/breakdown.txt 2>&1; echo "breakdown rc=$?" >> $O/summary.log
