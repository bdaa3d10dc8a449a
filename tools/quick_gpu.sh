# quick GPU check of a kernel change: sweep tests, cfg5 launch list, bench line
python -m pytest tests/test_sweep.py -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; tail -3 gpurun_out/q_tests.txt
python tools/one_solve.py 5 1 > gpurun_out/plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/q_launches_cfg5.csv python tools/one_solve.py 5 1 > gpurun_out/ncu_l5.log 2>&1
python tools/summarize_launches.py gpurun_out/q_launches_cfg5.csv > gpurun_out/q_launches_summary.txt; grep "sweep_reg\|one solve\|finalize_rows_kernel<18>   " gpurun_out/q_launches_summary.txt
python bench.py --no-cpu-baseline > gpurun_out/q_bench5.json 2> gpurun_out/q_bench5.err; python -c "
import json; d=json.load(open('gpurun_out/q_bench5.json')); print(d['value'], d['ms_per_step'], d['roofline']['combine_ms'], d['roofline']['frac'], d['parity'])"
