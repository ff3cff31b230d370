python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.json | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json | cut -c1-200
for ts in "8 2" "16 4" "32 8"; do set -- $ts; python bench.py --workload cfg5 --t $1 --s $2 --steps 2 --warmup 1 > gpurun_out/bench_cfg5_t$1.json 2>&1; tail -1 gpurun_out/bench_cfg5_t$1.json | cut -c1-200; done
timeout 900 python bench.py --workload cfg3 --steps 1 --warmup 1 --max-outer 6 --no-cpu --no-e2e --no-spmm-block > gpurun_out/bench_cfg3.json 2>&1; tail -1 gpurun_out/bench_cfg3.json | cut -c1-200
timeout 900 python bench.py --workload cfg4 --steps 1 --warmup 1 --max-outer 4 --no-cpu --no-e2e --no-spmm-block > gpurun_out/bench_cfg4.json 2>&1; tail -1 gpurun_out/bench_cfg4.json | cut -c1-200
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-spmm-block --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_sweep|k_spmm_grid|k_apply_tc|k_chol_fast" -s 200 -c 6 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_spmm_grid" -c 3 -o gpurun_out/prof_cfg5 python tools/spmm_micro.py --ops cfg5 --ts 8,16,32 --variants 2 --reps 1 > gpurun_out/ncu_c5.log 2>&1
