# Round-2 evidence (session 5): GPU suite, smoke, bench lines, TT-SVD, qr_bench, K4f ncu capture, 5b launch list.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/r02e_gputest.log 2>&1; tail -5 gpurun_out/r02e_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 3 5b; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02e_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02e_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['reasons'], d.get('phase_ms'))"
done
timeout 600 python tools/det3_time.py > gpurun_out/r02e_det3.json 2>&1; tail -1 gpurun_out/r02e_det3.json
timeout 300 python tools/qr_bench.py 40960 320 7040 110 25600 400 6400 400 2>&1 | grep "^qr " > gpurun_out/r02e_qr_bench.txt; cat gpurun_out/r02e_qr_bench.txt
echo done
