timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "batch" 2>&1 | tail -2
for f in 1 0; do TTR_KRP_BATCH=$f python bench.py --config 5a --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*'; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5a.csv python bench.py --config 5a --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l5a.csv 6
