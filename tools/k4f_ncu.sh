set -x
mkdir -p gpurun_out
TTR_QR_CQR=1 TTR_QR_DEV_SPEC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:cqr_panel_fused -s 12 -c 1 -f -o gpurun_out/k4f_panel python tools/qr_bench.py 40960 320 > gpurun_out/k4f_ncu.log 2>&1
tail -3 gpurun_out/k4f_ncu.log
ls -la gpurun_out/*.ncu-rep
