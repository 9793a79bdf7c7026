timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for f in 1 0; do for c in 1 2; do echo "small=$f cfg $c"; TTR_QR_SMALL_CTA=$f python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*'; done; done
