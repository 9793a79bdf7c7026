# CPU reference figures for BASELINE.md §5: 1 thread and all host threads
# (the oracle on its OpenBLAS backend; bench.py --impl reference = full config).
mkdir -p gpurun_out
for c in 1 3 5b; do
  timeout 1500 python bench.py --impl reference --config $c --cpu-threads 1 --steps 1 --warmup 0 2>/dev/null | tail -1 > gpurun_out/r02f_ref${c}_1thread.json
  python -c "import json; d=json.load(open('gpurun_out/r02f_ref${c}_1thread.json')); print('$c 1-thread', d['ms_per_step'], d['value'])"
done
for c in 1 3; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02f_ref${c}.json
  python -c "import json; d=json.load(open('gpurun_out/r02f_ref${c}.json')); print('$c all threads', d['ms_per_step'], d['value'], d['cpu_baseline']['cores'])"
done
timeout 900 python tools/det3_time.py --cpu > gpurun_out/r02f_det3_cpu.json 2>&1; tail -1 gpurun_out/r02f_det3_cpu.json
