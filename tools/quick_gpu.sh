for c in 4 3 2 1; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/q_bench$c.json 2>&1; done
