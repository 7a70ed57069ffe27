#!/bin/bash
# 2-GPU session: peer collectives parity (eager + graph), collective micro-bench, bench N=2.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for L in dp2 dp2z3; do
  ZB_COLLECTIVES=peer timeout 300 $TR --master-port 29611 scripts/mgpu_check.py $L > gpurun_out/peer2_$L.log 2>&1; echo "$L rc=$?" >> gpurun_out/peer2_summary.log
done
timeout 300 $TR --master-port 29612 scripts/coll_bench.py > gpurun_out/coll_bench_n2.log 2>&1; echo "coll rc=$?" >> gpurun_out/peer2_summary.log
timeout 400 $TR --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_peer_n2.log 2>&1; echo "bench rc=$?" >> gpurun_out/peer2_summary.log
