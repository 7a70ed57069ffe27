#!/bin/bash
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=gpurun_out/off4_summary.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_train_gpu.py -q -x > gpurun_out/off_tests.log 2>&1; echo "tests rc=$?" >> $S
for O in 0 1; do
  ZB_OFFLOAD=$O timeout 600 $TR --master-port 2969$O scripts/config_run.py xl_1+3 > gpurun_out/cfg_off$O.log 2>&1; echo "cfg off=$O rc=$?" >> $S
done
