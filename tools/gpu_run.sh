python -m pytest tests/test_gpu_parity.py -x -q -k "full_size_config" --durations=8 2>&1 | tail -8
