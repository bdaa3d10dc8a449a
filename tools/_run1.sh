set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/t1_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/t1_tests.txt
python bench.py > gpurun_out/t1_bench5.json 2> gpurun_out/t1_bench5.err
for c in 4 3 2 1; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/t1_bench$c.json 2>gpurun_out/t1_bench$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t1_launches5.csv python tools/one_solve.py 5 1 > gpurun_out/t1_ncu.log 2>&1
