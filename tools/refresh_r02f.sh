# Round-2 final evidence (session 5): GPU suite, smoke, bench lines of every config, reference arm,
# TT-SVD, TT-GMRES, QR timings, K4f ncu capture and trace, 5b / config-3 launch lists (every ncu under timeout).
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r02f_gputest.log 2>&1; tail -3 gpurun_out/r02f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 5a 1 2 3 4 5b; do  # 5a first: its eager multi-stream launches are host-bound and feel the host after a CPU-baseline leg
  sleep 5
  timeout 900 python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1
  tail -1 gpurun_out/bench_c$c.log > gpurun_out/r02f_bench$c.json
  python -c "import json; d=json.load(open('gpurun_out/r02f_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d['clocks']['reasons'], round(d['e2e']['value'],3), d['cpu_baseline']['value'])"
done
sleep 10
timeout 600 python tools/det3_time.py > gpurun_out/r02f_det3.json 2>&1; tail -1 gpurun_out/r02f_det3.json
timeout 600 python tools/gmres_time.py > gpurun_out/r02f_gmres.json 2>&1; tail -1 gpurun_out/r02f_gmres.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref5b.log 2>&1; tail -1 gpurun_out/ref5b.log > gpurun_out/r02f_ref5b.json; cut -c1-300 gpurun_out/r02f_ref5b.json
timeout 300 python tools/qr_bench.py 40960 320 7040 110 25600 400 6400 400 25600 16 1280 10 2>&1 | grep "^qr " > gpurun_out/r02f_qr_bench.txt; cat gpurun_out/r02f_qr_bench.txt
TTR_QR_DEV_SPEC=1 TTR_QR_TRACE=1 timeout 300 python tools/qr_bench.py 40960 320 2>&1 | grep -m 3 "cqr_panel_fused" > gpurun_out/r02f_k4f_trace.txt; cat gpurun_out/r02f_k4f_trace.txt
TTR_QR_DEV_SPEC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:cqr_panel_fused -s 12 -c 1 -f -o gpurun_out/r02f_k4f python tools/qr_bench.py 40960 320 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_5b_launches.csv python bench.py --config 5b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r02f_5b_launches.csv > gpurun_out/r02f_bench5b_launches.txt 2>&1; head -14 gpurun_out/r02f_bench5b_launches.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_3_launches.csv python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_table.py gpurun_out/r02f_3_launches.csv > gpurun_out/r02f_bench3_launches.txt 2>&1; head -12 gpurun_out/r02f_bench3_launches.txt
echo done
