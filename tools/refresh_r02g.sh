# after the speculation fixes (no speculation on rank-deficient bonds, counters restored on a rerun):
# GPU suite, 5b / config-3 bench lines, TT-SVD twice
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02f_gputest.log 2>&1; tail -3 gpurun_out/r02f_gputest.log
for c in 3 5b; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02f_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02f_bench$c.json')); print('$c', round(d['ms_per_step'],3), d['value'], d['config']['eager_ms_per_step'], d['config']['flops_per_step'], round(d['e2e']['value'],3), d['e2e']['ms_per_step'])"
done
for i in 1 2; do timeout 600 python tools/det3_time.py > gpurun_out/r02f_det3.json 2>&1; tail -1 gpurun_out/r02f_det3.json | cut -c1-150; done
echo done
