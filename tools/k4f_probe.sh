# K4f probe: correctness, per-phase trace, QR timings, 5b bench with/without the fused panels
set -x
mkdir -p gpurun_out
TTR_QR_CQR=1 timeout 600 python tools/qr_fused_check.py > gpurun_out/k4f_check.log 2>&1; tail -15 gpurun_out/k4f_check.log
TTR_QR_CQR=1 TTR_QR_DEV_SPEC=1 TTR_QR_TRACE=1 timeout 300 python tools/qr_bench.py 40960 320 2>&1 | grep -m 12 "cqr_panel_fused"
for v in 0 1; do
  TTR_QR_CQR=$v TTR_QR_DEV_SPEC=1 timeout 300 python tools/qr_bench.py 40960 320 7040 110 20480 320 2>&1 | grep "^qr "
done
TTR_GEMM_LTFOLD=0 timeout 300 python tools/qr_bench.py 40960 320 2>&1 | grep "^qr "
for v in 0 1; do
  TTR_QR_CQR=$v timeout 900 python bench.py --config 5b --no-cpu-baseline --no-e2e > gpurun_out/k4f_5b_cqr$v.log 2>&1
  tail -1 gpurun_out/k4f_5b_cqr$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('5b cqr$v', d['ms_per_step'], d['phase_ms'])"
done
echo done
