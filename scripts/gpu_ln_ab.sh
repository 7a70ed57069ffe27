#!/bin/bash
for i in 1 2; do
python scripts/ln_bench.py paper_2507_10392_b200/libzorse_b200_old.so
python scripts/ln_bench.py
done
