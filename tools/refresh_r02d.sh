# Round-2 evidence (session 4): GPU suite, smoke, bench lines, TT-SVD,
# TT-GMRES criterion 8, K4e ncu capture, 5a launch list.
set -x
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02d_gputest.log 2>&1; tail -3 gpurun_out/r02d_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 4 5a 5b; do
  python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02d_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02d_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['reasons'])"
done
python tools/det3_time.py > gpurun_out/r02d_det3.json 2>&1; tail -1 gpurun_out/r02d_det3.json
python tools/gmres_time.py --cpu > gpurun_out/r02d_gmres.json 2>&1; tail -1 gpurun_out/r02d_gmres.json
ncu --set full --import-source on --clock-control none -k regex:cholqr_small -s 10 -c 1 -o gpurun_out/r02d_cqr python bench.py --config 5a --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_5a_launches.csv python bench.py --config 5a --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
