bash tools/ab_run.sh 5 7 r1 v0r0 v0r1 v2r1 v2r0 > gpurun_out/ab3_cfg5.txt 2>&1
