python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo tests_rc=$? >> gpurun_out/q_tests.txt
python tools/sweep.py 5 --reps 5 --levels > gpurun_out/q_levels5.txt 2>&1
for c in 5 4 3 2; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/q_bench$c.json 2>&1; done
