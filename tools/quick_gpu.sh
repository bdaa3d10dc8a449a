python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo tests_rc=$? >> gpurun_out/q_tests.txt
python tools/batch_throughput.py gpurun_out/q_batch.json > gpurun_out/q_batch.txt 2>&1
for c in 5 2; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/q_bench$c.json 2>&1; done
