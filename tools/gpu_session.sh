mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "cholesky or chol" > gpurun_out/s_test.log 2>&1; tail -3 gpurun_out/s_test.log
python tools/qr_bench.py 7040 110 6400 100 12800 120 2>&1 | grep -v torch
TTR_QR_CHOL=1 timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/s_c3.log 2>&1
tail -1 gpurun_out/s_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 chol', round(d['ms_per_step'],3), d.get('phase_ms'))"
