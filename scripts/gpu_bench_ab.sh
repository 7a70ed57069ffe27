#!/bin/bash
# same-box A/B of two library builds through the full bench (N=1)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in old new; do
    lib=paper_2507_10392_b200/libzorse_b200.so; [ $v = old ] && lib=paper_2507_10392_b200/libzorse_b200_old.so
    python scripts/bench_ab.py $lib --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
