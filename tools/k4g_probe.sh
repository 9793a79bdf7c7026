set -x
mkdir -p gpurun_out
timeout 600 python tools/qr_fused_check.py > gpurun_out/k4f_check.log 2>&1; tail -16 gpurun_out/k4f_check.log
TTR_QR_DEV_SPEC=1 timeout 300 python tools/qr_bench.py 25600 16 12800 16 1280 10 2>&1 | grep "^qr "
TTR_QR_CQR=0 TTR_QR_DEV_SPEC=1 timeout 300 python tools/qr_bench.py 25600 16 12800 16 1280 10 2>&1 | grep "^qr "
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "adaptive or sum or gmres or det or qr" > gpurun_out/k4g_tests.log 2>&1; tail -5 gpurun_out/k4g_tests.log
for c in 2 4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/k4g_c$c.log 2>&1
  tail -1 gpurun_out/k4g_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['config'].get('eager_ms_per_step'), d['config'].get('plan_rerecords'), d['config'].get('output_ranks'))"
done
echo done
