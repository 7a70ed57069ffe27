#!/bin/bash
# A/B/C of attention builds on one box: bash scripts/gpu_attn_multi.sh LIB1 LIB2 ...
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k attention -p no:cacheprovider 2>&1 | tail -n 1
for i in 1 2; do
  for lib in "$@"; do
    python scripts/bench_attn.py "$lib" > gpurun_out/attn_multi.jsonl
    python -c "
import json,sys
r=[json.loads(l) for l in open('gpurun_out/attn_multi.jsonl')]
print('%-40s' % sys.argv[1].split('/')[-1], ' '.join('%s f%d b%d' % ('x'.join(map(str,x['shape'][::2][:1]+[x['shape'][3]])), x['fwd_tflops'], x['bwd_tflops(2.5x fwd flops)']) for x in r))" "$lib"
  done
done
