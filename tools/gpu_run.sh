for c in 1 2 4 5a; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench$c.json 2> gpurun_out/bench$c.err; echo "cfg $c rc=$?"; tail -2 gpurun_out/bench$c.err
done
