set -x
mkdir -p gpurun_out
TTR_QR_CQR=1 timeout 600 python tools/qr_fused_check.py > gpurun_out/k4f_check.log 2>&1; tail -12 gpurun_out/k4f_check.log
TTR_QR_CQR=1 TTR_QR_DEV_SPEC=1 TTR_QR_TRACE=1 timeout 300 python tools/qr_bench.py 40960 320 2>&1 | grep -m 3 "cqr_panel_fused"
TTR_QR_CQR=1 TTR_QR_DEV_SPEC=1 TTR_QR_TRACE=1 timeout 300 python tools/qr_bench.py 7040 110 2>&1 | grep -m 4 "cqr_panel_fused"
TTR_QR_CQR=1 TTR_QR_DEV_SPEC=1 timeout 300 python tools/qr_bench.py 40960 320 7040 110 20480 320 12800 64 2>&1 | grep "^qr "
TTR_QR_CQR=1 timeout 900 python bench.py --config 5b --no-cpu-baseline --no-e2e > gpurun_out/k4f_5b_cqr1.log 2>&1
tail -1 gpurun_out/k4f_5b_cqr1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('5b cqr1', d['ms_per_step'], d['phase_ms'])"
TTR_QR_CQR=1 timeout 900 python bench.py --config 3 --no-cpu-baseline --no-e2e > gpurun_out/k4f_3_cqr1.log 2>&1
tail -1 gpurun_out/k4f_3_cqr1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('3 cqr1', d['ms_per_step'], d.get('phase_ms'))"
echo done
