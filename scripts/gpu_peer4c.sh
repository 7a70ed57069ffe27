#!/bin/bash
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/peer4c_summary.log
for L in dp4z3 pp1+3; do
  timeout 300 $TR --master-port 29641 scripts/mgpu_check.py $L > gpurun_out/peer4c_$L.log 2>&1; echo "$L rc=$?" >> $S
done
for i in 1 2 3 4; do
timeout 300 $TR --master-port 2965$i bench.py --gpus 4 --steps 60 --warmup 3 > gpurun_out/b4c_$i.log 2>&1; echo "bench $i rc=$?" >> $S
done
