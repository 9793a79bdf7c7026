# Regenerate the per-config bench lines (profiles/r01_bench{1,2,3,4,5a}.json) on the GPU box
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in 1 2 3 4 5a; do python bench.py --config $c > gpurun_out/bench_c$c.log 2>&1; tail -1 gpurun_out/bench_c$c.log > gpurun_out/r01_bench$c.json; python -c "import json; d=json.load(open('gpurun_out/r01_bench$c.json')); print('$c', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), d.get('ranks_identical'), d['clocks']['reasons'])"; done
python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-300
