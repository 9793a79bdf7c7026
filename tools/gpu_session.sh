set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "cholesky or fixed_krp or plan or thin_qr" > gpurun_out/t1.log 2>&1; grep -E "^E |passed|failed" gpurun_out/t1.log | head
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/c3.json; python -c "import json; d=json.load(open('gpurun_out/c3.json')); print(d['ms_per_step'], d['phase_ms'])"
TTR_QR_CHOL=1 timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/c3c.json; python -c "import json; d=json.load(open('gpurun_out/c3c.json')); print(d['ms_per_step'], d['phase_ms'])"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/c5b.json; python -c "import json; d=json.load(open('gpurun_out/c5b.json')); print(d['ms_per_step'], d['phase_ms'])"
