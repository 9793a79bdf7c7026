set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "batch" > gpurun_out/t1.log 2>&1; grep -E "^E |passed|failed" gpurun_out/t1.log | head
for g in 1 2 4 8; do TTR_BATCH_GROUPS=$g timeout 300 python bench.py --config 5a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/c5a_$g.json; python -c "import json; d=json.load(open('gpurun_out/c5a_$g.json')); print($g, d['ms_per_step'], d['phase_ms'])"; done
