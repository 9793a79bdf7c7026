timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sum or adaptive or counters" 2>&1 | tail -2
python tools/config_bench.py 4sum 3sum 2>&1 | tail -3
