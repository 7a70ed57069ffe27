#!/bin/bash
# One GPU session: tests, gemm micro-bench in both CTA modes, bench.
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.log
ZB_GEMM_CTAS=1 timeout 300 python scripts/bench_gemm.py > gpurun_out/gemm_1cta.log 2>&1
ZB_GEMM_CTAS=2 timeout 300 python scripts/bench_gemm.py > gpurun_out/gemm_2cta.log 2>&1
timeout 300 python scripts/bench_gemm.py > gpurun_out/gemm_auto.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gpu_tests.log
