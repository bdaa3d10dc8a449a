# round-2 (row sweep) profile set: run on the GPU box from the repo root
set -x
O=gpurun_out/prof; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/r2s_gpu_tests.txt 2>&1; tail -2 $O/r2s_gpu_tests.txt
python tools/one_solve.py 5 1 > $O/plain.log 2>&1 || exit 1
for c in 5 4 3 2; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/r2s_launches_cfg$c.csv python tools/one_solve.py $c 1 > $O/ncu_l$c.log 2>&1
python tools/summarize_launches.py $O/r2s_launches_cfg$c.csv > $O/r2s_launches_cfg${c}_summary.txt
python tools/traffic.py $O/r2s_launches_cfg$c.csv $c > $O/traffic_cfg$c.json
done
cap() { # name regex skip
ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $O/$1 -f python tools/one_solve.py 5 1 > $O/ncu_$1.log 2>&1
python tools/ncu_summary.py $O/$1.ncu-rep "$1 (cfg5)" > $O/$1.txt
}
# ncu matches the base kernel name: the sweep launches of a cfg5 solve are, in
# order, sweep_reg_kernel <5,0> <9,0> <17,0> (warp groups), two sweep_reg_small_kernel
# (CTA groups of 128 / 256 threads, h = 1024 / 2048) and sweep_reg_kernel <9,1> for
# h = 4096, h = 8192 (half-size pass, then the flagged pass) and the root
cap r2s_ncu_sweep_warp5 "sweep_reg_kernel" 0
cap r2s_ncu_sweep_warp9 "sweep_reg_kernel" 1
cap r2s_ncu_sweep_warp17 "sweep_reg_kernel" 2
cap r2s_ncu_sweep_cta_h1024 "sweep_reg_small_kernel" 0
cap r2s_ncu_sweep_cta_h4096 "sweep_reg_kernel" 3
cap r2s_ncu_sweep_cta_h8192 "sweep_reg_kernel" 4
cap r2s_ncu_sweep_cta_top "sweep_reg_kernel" 6
cap r2s_ncu_skeleton "^skeleton_kernel" 3
cap r2s_ncu_finalize "finalize_rows_kernel" 4
cap r2s_ncu_narrow8 "narrow_combine_kernel" 2
cap r2s_ncu_roll "narrow32_roll_kernel" 0
python tools/issue_json.py $O/r2s_launches_cfg5_summary.txt "sweep_reg_kernel<5"=$O/r2s_ncu_sweep_warp5.txt "sweep_reg_kernel<9, 0"=$O/r2s_ncu_sweep_warp9.txt "sweep_reg_kernel<17"=$O/r2s_ncu_sweep_warp17.txt "sweep_reg_small_kernel"=$O/r2s_ncu_sweep_cta_h1024.txt "sweep_reg_kernel<9, 1"=$O/r2s_ncu_sweep_cta_h4096.txt "skeleton_kernel"=$O/r2s_ncu_skeleton.txt "finalize_rows"=$O/r2s_ncu_finalize.txt "narrow_combine_kernel"=$O/r2s_ncu_narrow8.txt "narrow32_roll"=$O/r2s_ncu_roll.txt > $O/issue_cfg5.json
cat $O/issue_cfg5.json | tail -5
# the bench lines embed profiles/traffic_cfg*.json and profiles/issue_cfg5.json: install the fresh ones first
cp $O/traffic_cfg*.json $O/issue_cfg5.json profiles/
python bench.py > $O/r2s_bench_cfg5.json 2> $O/bench5.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/r2s_bench_reference_cfg5.json 2> $O/ref.err
for c in 4 3 2; do python bench.py --config $c --steps 20 > $O/r2s_bench_cfg$c.json 2> $O/bench$c.err; done
python bench.py --config 1 --steps 400 --warmup 20 > $O/r2s_bench_cfg1.json 2> $O/bench1.err
python -c "import __graft_entry__ as g; g.smoke()"
python tools/batch_throughput.py > $O/r2s_batch_throughput.json 2>&1
python tools/fuzz_parity.py 240 2024 > $O/r2s_fuzz.txt 2>&1; tail -1 $O/r2s_fuzz.txt
rm -f $O/*.ncu-rep
