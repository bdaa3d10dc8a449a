run() { echo "== $*"; env "$@" python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['combine_ms'], d['parity'])"; }
run A=1
run LCSG_SKEL_STRIDE_H7=128 LCSG_SKEL_STRIDE_H8=128 LCSG_SKEL_STRIDE_H9=128
run LCSG_SKEL_STRIDE_H7=128 LCSG_SKEL_STRIDE_H8=128 LCSG_SKEL_STRIDE_H9=128 LCSG_SKEL_STRIDE_H10=128 LCSG_SKEL_STRIDE_H11=128
run LCSG_SKEL_STRIDE_H13=32 LCSG_SKEL_STRIDE_H14=32
run LCSG_SKEL_STRIDE_H14=32
run LCSG_SWEEP_GN_MAX=512
run LCSG_SKEL_STRIDE_H7=32 LCSG_SKEL_STRIDE_H8=32
