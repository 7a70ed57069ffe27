#!/bin/bash
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/peer4d_summary.log
CUDA_VISIBLE_DEVICES=0 timeout 200 python scripts/bench_attn.py > gpurun_out/p4d_attn.log 2>&1; echo "attn rc=$?" >> $S
for i in 1 2; do
ZB_PEER_AG=sm timeout 200 $TR --master-port 2966$i bench.py --gpus 4 --steps 60 --warmup 3 > gpurun_out/b4d_sm$i.log 2>&1; echo "bench sm $i rc=$?" >> $S
done
for i in 1 2; do
timeout 200 $TR --master-port 2967$i bench.py --gpus 4 --steps 60 --warmup 3 > gpurun_out/b4d_ce$i.log 2>&1; echo "bench ce $i rc=$?" >> $S
done
