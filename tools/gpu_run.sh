python -m pytest tests/test_gpu_parity.py -x -q -k "qr or fixed or config3" 2>&1 | tail -2
python tools/qr_bench.py 40960 320 7040 110 2>&1 | grep -v torch
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*\|"phase_ms": {[^}]*}'
