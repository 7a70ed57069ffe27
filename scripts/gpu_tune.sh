#!/bin/bash
mkdir -p gpurun_out
python scripts/tune_gemm.py --out gpurun_out/gemm_tune_cache.txt > gpurun_out/tune.log 2>&1; tail -3 gpurun_out/tune.log
cp gpurun_out/gemm_tune_cache.txt paper_2507_10392_b200/gemm_tune_cache.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
python -c "import json; d=json.load(open('gpurun_out/bench_n1.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"
