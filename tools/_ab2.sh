LCSG_LIB_PATH=paper_2309_09072_b200/lib/ab/t1.so python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or strides or digests" > gpurun_out/t16_tests.txt 2>&1; echo rc=$? >> gpurun_out/t16_tests.txt
for v in t0 t1 t0 t1; do echo "== $v"; LCSG_LIB_PATH=paper_2309_09072_b200/lib/ab/$v.so LCSG_GRAPH=0 python tools/sweep.py 5 --reps 3 2>&1 | grep -E "combine |rror"; done > gpurun_out/ab12.txt 2>&1
echo "== t1 carveouts" >> gpurun_out/ab12.txt
LCSG_LIB_PATH=paper_2309_09072_b200/lib/ab/t1.so LCSG_GRAPH=0 python tools/sweep.py 5 --reps 3 LCSG_FINE_CARVEOUT=64 LCSG_FINE_CARVEOUT=80 LCSG_FINE_CARVEOUT=56 2>&1 | grep -E "combine |rror" >> gpurun_out/ab12.txt
for v in t0 t1; do echo "== $v cfg4"; LCSG_LIB_PATH=paper_2309_09072_b200/lib/ab/$v.so LCSG_GRAPH=0 python tools/sweep.py 4 --reps 3 2>&1 | grep -E "combine |rror"; done >> gpurun_out/ab12.txt 2>&1
