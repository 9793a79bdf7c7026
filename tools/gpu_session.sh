set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "batch" > gpurun_out/t1.log 2>&1; grep -E "^E |passed|failed" gpurun_out/t1.log | head
for v in 0 1; do TTR_LR_QR=$v timeout 300 python bench.py --config 5a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/c5a_$v.json; python -c "import json; d=json.load(open('gpurun_out/c5a_$v.json')); print($v, d['ms_per_step'], d['phase_ms'], d['roofline']['achieved'])"; done
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l5a.csv python bench.py --config 5a --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/l5a.csv 10
