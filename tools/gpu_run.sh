timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "adaptive or counters or full_size_config or edge or zero or cli or compression" 2>&1 | tail -2
for c in 2 4; do python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*\|"gpu_launches_per_step": [0-9]*' | tr '\n' ' '; echo; done
