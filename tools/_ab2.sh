python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or window or digests or reference" > gpurun_out/tma_tests.txt 2>&1; echo rc=$? >> gpurun_out/tma_tests.txt
for v in tma0 tma1 tma0 tma1; do echo "== $v"; LCSG_LIB_PATH=paper_2309_09072_b200/lib/ab/$v.so python tools/sweep.py 5 --reps 3 --levels 2>&1 | grep -E "combine |narrow|rror"; done > gpurun_out/ab6.txt 2>&1
