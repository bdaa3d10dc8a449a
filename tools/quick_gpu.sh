python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.txt 2>&1; echo tests_rc=$? >> gpurun_out/q_tests.txt
for c in 5 4 3 2 1; do python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/q_bench$c.json 2>&1; done
LCSG_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --config 3 > gpurun_out/q_dist.json 2> gpurun_out/q_dist.err
