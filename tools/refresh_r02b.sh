# Round-2 (session 3) evidence on the GPU box: GPU suite, smoke, every config's
# bench line, TT-SVD timing, the 5b reference arm (bounded), launch lists.
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02b_gputest.log 2>&1; tail -3 gpurun_out/r02b_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 4 5a 5b; do
  python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02b_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02b_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['reasons'], d.get('e2e') and round(d['e2e'].get('ms_per_step', 0) or 0, 2), d.get('cpu_baseline') and d['cpu_baseline'].get('value'))"
done
python tools/det3_time.py > gpurun_out/r02b_det3.json 2>&1; tail -1 gpurun_out/r02b_det3.json
python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 > gpurun_out/r02b_ref5b.json; head -c 400 gpurun_out/r02b_ref5b.json; echo
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches5b.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r02b_launches5b.csv 12
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_det3.csv python tools/det3_time.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r02b_launches_det3.csv 10
echo done
