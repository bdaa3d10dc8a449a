python tools/one_solve.py 5 1 > gpurun_out/plain.log 2>&1 || exit 1
for c in 5 4 3 2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches_cfg$c.csv python tools/one_solve.py $c 1 > gpurun_out/ncu_l$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:narrow_combine_kernel -s 2 -c 1 -o gpurun_out/r2_narrow8 python tools/one_solve.py 5 1 > gpurun_out/ncu_n8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:narrow32_roll -c 1 -o gpurun_out/r2_roll python tools/one_solve.py 5 1 > gpurun_out/ncu_roll.log 2>&1
