mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "batched or cholesky or config5a" > gpurun_out/s_test.log 2>&1; tail -3 gpurun_out/s_test.log
timeout 300 python bench.py --config 5a --no-cpu-baseline --no-e2e > gpurun_out/s_5a.log 2>&1
tail -1 gpurun_out/s_5a.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), d['phase_ms'])"
