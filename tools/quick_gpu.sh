python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo tests_rc=$? >> gpurun_out/q_tests.txt
for c in 5 4 3 2 1; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/q_bench$c.json 2>&1; done
