run() { echo "== $*"; env "$@" python tools/one_solve.py 5 1 > /dev/null 2>&1
env "$@" ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv python tools/one_solve.py 5 1 > /dev/null 2>&1
python tools/summarize_launches.py gpurun_out/ab.csv | grep "sweep_reg_kernel<9, 1.*grid\|one solve"; }
run LCSG_SWEEP_SMALL_CAP=0
run LCSG_SWEEP_SMALL_CAP=1
run LCSG_LIB_PATH=$PWD/paper_2309_09072_b200/lib/variants/libmb6.so
