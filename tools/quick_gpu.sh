set -x
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "strides or variants or digests or window or cta_wide or reference_trees" > gpurun_out/q_tests.txt 2>&1; echo tests_rc=$? >> gpurun_out/q_tests.txt
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/q_bench5.json 2>&1
python bench.py --no-cpu-baseline --config 4 --steps 10 > gpurun_out/q_bench4.json 2>&1
python bench.py --no-cpu-baseline --config 3 --steps 10 > gpurun_out/q_bench3.json 2>&1
