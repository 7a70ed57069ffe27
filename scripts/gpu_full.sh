#!/bin/bash
# Full single-GPU validation + bench + launch list.
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --impl reference > gpurun_out/bench_ref.log 2>&1
python scripts/profile_step.py 2 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python scripts/profile_step.py 2 > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -1 gpurun_out/smoke.log
