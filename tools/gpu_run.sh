python bench.py --config 5a --steps 5 --warmup 3 > gpurun_out/w.json 2>gpurun_out/w.err; grep -o '"ms_per_step": [0-9.]*' gpurun_out/w.json
python -m pytest tests/test_gpu_parity.py -x -q -k "batch" 2>&1 | tail -2
