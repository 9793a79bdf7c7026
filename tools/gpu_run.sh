for i in 1 2; do python bench.py --config 2 > gpurun_out/h_bench2.json 2> gpurun_out/h_bench2.err; grep -o '"ms_per_step": [0-9.]*\|"clocks": {[^}]*}' gpurun_out/h_bench2.json | head -2; done
python bench.py --config 4 > gpurun_out/h_bench4.json 2> gpurun_out/h_bench4.err; grep -o '"ms_per_step": [0-9.]*\|"clocks": {[^}]*}' gpurun_out/h_bench4.json | head -2
python bench.py > gpurun_out/h_bench5b.json 2> gpurun_out/h_bench5b.err; grep -o '"ms_per_step": [0-9.]*\|"clocks": {[^}]*}' gpurun_out/h_bench5b.json | head -2
