#!/bin/bash
# Planner loop on B200: measure layer timings -> cluster profile -> plan_training ->
# execute -> report estimate vs simulated vs measured (profiles/r02_report_*).
mkdir -p gpurun_out profiles
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python scripts/profile_layers.py gpt2-small-124m 4 > gpurun_out/r02_measured_profile_gpt2s_n4.json 2> gpurun_out/profile.err
timeout 600 $TR --nproc-per-node 4 --master-port 29531 scripts/report.py --out gpurun_out --profile gpurun_out/r02_measured_profile_gpt2s_n4.json --global-batch 32 --tag measured_profile_gpt2s_n4 > gpurun_out/report_profile.log 2>&1
timeout 600 $TR --nproc-per-node 4 --master-port 29532 scripts/report.py --out gpurun_out --tag bench_n4 > gpurun_out/report_bench4.log 2>&1
timeout 600 python scripts/report.py --out gpurun_out --tag bench_n1 > gpurun_out/report_bench1.log 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29533 scripts/report.py --out gpurun_out --config xl_1+3 --tag xl_1+3_n4 > gpurun_out/report_xl.log 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29534 scripts/report.py --out gpurun_out --config llama13b_plan4 --steps 3 --tag llama13b_plan4_n4 > gpurun_out/report_13b.log 2>&1
timeout 900 $TR --nproc-per-node 4 --master-port 29535 scripts/report.py --out gpurun_out --config llama7b_2x2 --steps 3 --tag llama7b_2x2_n4 > gpurun_out/report_7b.log 2>&1
grep -h "latency\|GB\|report" gpurun_out/report_*.log | grep -v Warning | head -40
