# CPU reference figures for BASELINE.md §5: 1 thread and all host threads
# (the oracle on its OpenBLAS backend; bench.py --impl reference = full config).
for c in 1 3 5b; do
  python bench.py --impl reference --config $c --cpu-threads 1 --steps 1 --warmup 0 2>/dev/null | tail -1 > gpurun_out/r02_ref${c}_1thread.json
  python -c "import json; d=json.load(open('gpurun_out/r02_ref${c}_1thread.json')); print('$c 1-thread', d['ms_per_step'], d['value'])"
done
python bench.py --impl reference --config 1 --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02_ref1.json
python tools/det3_time.py --cpu > gpurun_out/r02_det3.json 2>&1; tail -1 gpurun_out/r02_det3.json
