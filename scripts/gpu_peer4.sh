#!/bin/bash
# 4-GPU session: peer collectives parity on every 4-rank layout (graph replay),
# collective micro-bench, bench N=4 (peer and NCCL), full-size config runs.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/peer4_summary.log
for L in pp1+3 dp4z3 pp2x2 llama1f1b2x2 xl1+3; do
  timeout 300 $TR --master-port 29621 scripts/mgpu_check.py $L > gpurun_out/peer4_$L.log 2>&1; echo "$L rc=$?" >> $S
done
timeout 300 $TR --master-port 29622 scripts/coll_bench.py > gpurun_out/coll_bench_n4.log 2>&1; echo "coll rc=$?" >> $S
timeout 400 $TR --master-port 29623 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_peer_n4.log 2>&1; echo "bench peer rc=$?" >> $S
timeout 400 $TR --master-port 29624 bench.py --gpus 4 --steps 10 --warmup 3 --collectives nccl > gpurun_out/bench_nccl_n4.log 2>&1; echo "bench nccl rc=$?" >> $S
for C in xl_1+3 llama7b_2x2; do
  timeout 600 $TR --master-port 29625 scripts/config_run.py $C > gpurun_out/cfg_peer_$C.log 2>&1; echo "cfg $C rc=$?" >> $S
done
