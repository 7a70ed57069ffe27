#!/bin/bash
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/peer4b_summary.log
timeout 300 $TR --master-port 29631 bench.py --gpus 4 --steps 10 --warmup 3 --eager > gpurun_out/b4_eager.log 2>&1; echo "eager rc=$?" >> $S
ZB_PEER_AG=sm timeout 300 $TR --master-port 29632 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b4_sm.log 2>&1; echo "graph sm rc=$?" >> $S
timeout 300 $TR --master-port 29633 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/b4_ce.log 2>&1; echo "graph ce rc=$?" >> $S
