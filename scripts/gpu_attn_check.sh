#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k attention -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1; tail -n 3 gpurun_out/attn_tests.log
timeout 300 python scripts/bench_attn.py
