#!/bin/bash
# 4-GPU round-end evidence: parity on every layout (peer collectives, CUDA graph),
# collective micro-bench, bench at N=2 and N=4 (both arms), full-size configs.
O=gpurun_out/r1b_final4c
mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for L in pp1+3 dp4z3 pp2x2 llama1f1b2x2 xl1+3; do
  timeout 300 $TR --nproc-per-node 4 --master-port 29701 scripts/mgpu_check.py $L > $O/parity_$L.log 2>&1; echo "$L rc=$?" >> $O/summary.log
done
timeout 300 $TR --nproc-per-node 4 --master-port 29702 scripts/coll_bench.py > $O/coll_n4.log 2>&1; echo "coll rc=$?" >> $O/summary.log
for N in 2 4; do
  timeout 400 $TR --nproc-per-node $N --master-port 2971$N bench.py --gpus $N --steps 10 --warmup 3 > $O/bench_n$N.log 2>&1; echo "bench n$N rc=$?" >> $O/summary.log
  timeout 400 $TR --nproc-per-node $N --master-port 2972$N bench.py --gpus $N --steps 3 --warmup 3 --impl reference > $O/bench_ref_n$N.log 2>&1; echo "ref n$N rc=$?" >> $O/summary.log
done
for C in xl_1+3 llama7b_2x2; do
  timeout 600 $TR --nproc-per-node 4 --master-port 29731 scripts/config_run.py $C > $O/cfg_$C.log 2>&1; echo "cfg $C rc=$?" >> $O/summary.log
done
