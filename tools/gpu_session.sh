set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "cholesky" > gpurun_out/t1.log 2>&1; grep -E "^E |passed|failed" gpurun_out/t1.log | head
timeout 300 python tools/qr_bench.py 40960 320 7040 110 6400 400 2>&1 | grep -v "^ *$" | head -30
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qrc.csv python tools/qr_chol_probe.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/qrc.csv 20
TTR_QR_DEBUG=1 timeout 300 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -v "^{" | tail -5
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c3.json; python -c "import json; d=json.load(open('gpurun_out/c3.json')); print(d['ms_per_step'], d['phase_ms'])"
TTR_QR_DEBUG=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -v "^{" | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/c5b.json; python -c "import json; d=json.load(open('gpurun_out/c5b.json')); print(d['ms_per_step'], d['phase_ms'])"
