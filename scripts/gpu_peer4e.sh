#!/bin/bash
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/peer4e_summary.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_kernels_gpu.py tests/test_train_gpu.py -q -x > gpurun_out/p4e_tests.log 2>&1; echo "tests rc=$?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 200 python scripts/bench_attn.py > gpurun_out/p4e_attn.log 2>&1; echo "attn rc=$?" >> $S
for i in 1 2 3 4; do
timeout 200 $TR --master-port 2968$i bench.py --gpus 4 --steps 60 --warmup 3 > gpurun_out/b4e_$i.log 2>&1; echo "bench $i rc=$?" >> $S
done
