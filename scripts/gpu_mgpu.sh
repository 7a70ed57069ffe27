#!/bin/bash
# Multi-GPU round check on a 4-GPU box: per-tensor parity layouts, BASELINE config
# layouts with memory vs the plan's estimate, bench N=2/4.  Output -> gpurun_out/
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for L in dp2:2 dp2z3:2 pp2:2 cfg1_tiny:3 pp1+3:4 dp4z3:4 pp2x2:4 llama1f1b2x2:4 xl1+3:4; do
  name=${L%%:*}; n=${L##*:}
  timeout 600 $TR --nproc-per-node $n --master-port 29511 scripts/mgpu_check.py $name >> gpurun_out/mgpu_parity.jsonl 2>> gpurun_out/mgpu_parity.err
  echo "$name rc=$?" >> gpurun_out/mgpu_parity.rc
done
for R in xl_1+3 llama7b_2x2 llama13b_plan4; do
  timeout 900 $TR --nproc-per-node 4 --master-port 29512 scripts/config_run.py $R 3 >> gpurun_out/config_runs.jsonl 2>> gpurun_out/config_runs.err
  echo "$R rc=$?" >> gpurun_out/config_runs.rc
done
timeout 600 $TR --nproc-per-node 2 --master-port 29513 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29514 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
cat gpurun_out/mgpu_parity.rc gpurun_out/config_runs.rc
