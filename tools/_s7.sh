python tools/one_solve.py 5 1 > gpurun_out/plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sweep_reg_kernel -c 1 -o gpurun_out/s7_reg5 -f python tools/one_solve.py 5 1 > gpurun_out/ncu_a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_reg_kernel -s 3 -c 1 -o gpurun_out/s7_reg9m -f python tools/one_solve.py 5 1 > gpurun_out/ncu_b.log 2>&1
python tools/ncu_summary.py gpurun_out/s7_reg5.ncu-rep "reg5" > gpurun_out/s7_reg5.txt
python tools/ncu_summary.py gpurun_out/s7_reg9m.ncu-rep "reg9m" > gpurun_out/s7_reg9m.txt
python tools/ncu_lines.py gpurun_out/s7_reg5.ncu-rep 45 > gpurun_out/s7_reg5_lines.txt
python tools/ncu_lines.py gpurun_out/s7_reg9m.ncu-rep 45 > gpurun_out/s7_reg9m_lines.txt
cat gpurun_out/s7_reg5.txt gpurun_out/s7_reg5_lines.txt
