set -x
mkdir -p gpurun_out
TTR_QR_DEV_SPEC=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr5b_launches.csv python tools/qr_once.py 40960 320 > gpurun_out/qr_once.log 2>&1
tail -2 gpurun_out/qr_once.log
python tools/launch_table.py gpurun_out/qr5b_launches.csv > gpurun_out/qr5b_launches.txt 2>&1; cat gpurun_out/qr5b_launches.txt
