#!/bin/bash
# same-box A/B of the whole tree: ab_old/ (a worktree of the previous commit, built) vs this one
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in old new; do
    b=bench.py; [ $v = old ] && b=ab_old/bench.py
    python $b --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['e2e']['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
done
