#!/bin/bash
# One call of every kernel family + a smoke step (scripts/sanitize_kernels.py).
# compute-sanitizer itself is closed on the GPU pool (profiles/r02_compute_sanitizer_pool_closed.txt),
# so this runs plain; bounds are asserted on the host side of every C-ABI entry point.
mkdir -p gpurun_out
python scripts/sanitize_kernels.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
tail -n 3 gpurun_out/sanitize_plain.log
