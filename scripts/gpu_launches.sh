mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 > gpurun_out/ll_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ll_ncu.log 2>&1
echo rc=$?
python scripts/launch_summary.py gpurun_out/launches_r02.csv 4 | head -40
