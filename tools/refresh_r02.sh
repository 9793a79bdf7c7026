# Round-2 evidence on the GPU box: GPU suite, smoke, every config's bench line,
# the 5b reference arm (bounded steps), the 5b launch list.
set -x
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02_gputest.log 2>&1; tail -3 gpurun_out/r02_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 4 5a 5b; do
  python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d.get('ranks_identical'), d['clocks']['reasons'], d.get('cpu_baseline',{}) and d['cpu_baseline'].get('value'))"
done
python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02_ref5b.json
python bench.py --impl reference --config 3 --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02_ref3.json
python bench.py --local-ranks 2 --steps 3 --warmup 1 --no-e2e 2>/dev/null | tail -1 > gpurun_out/r02_bench5b_local2.json
python bench.py --local-ranks 8 --steps 2 --warmup 1 --no-e2e 2>/dev/null | tail -1 > gpurun_out/r02_bench5b_local8.json
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches5b.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
