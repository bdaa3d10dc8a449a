python tools/one_solve.py 5 1 > gpurun_out/plain.log 2>&1 || exit 1
for spec in "0 reg5" "4 reg9m_h2048" "7 reg9m_top"; do
set -- $spec
ncu --set full --clock-control none --import-source on -k regex:sweep_reg_kernel -s $1 -c 1 -o gpurun_out/s7_$2 -f python tools/one_solve.py 5 1 > gpurun_out/ncu_$2.log 2>&1
python tools/ncu_summary.py gpurun_out/s7_$2.ncu-rep "$2" > gpurun_out/s7_$2.txt
python tools/ncu_lines.py gpurun_out/s7_$2.ncu-rep 40 > gpurun_out/s7_$2_lines.txt
done
cat gpurun_out/s7_reg5.txt gpurun_out/s7_reg5_lines.txt
