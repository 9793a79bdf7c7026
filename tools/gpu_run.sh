TTR_CQR_TRACE=1 python tools/qr_bench.py 40960 32 2>&1 | grep -a -A6 cqr | tail -8
