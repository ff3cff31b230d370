# round deliverables: full bench line (cpu_baseline + e2e), reference arm, launch list, ncu full of the top kernels
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -1 gpurun_out/bench_full.json
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_sweep|k_spmm_gram|k_apply_tc" -s 300 -c 8 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_f.log 2>&1
tail -1 gpurun_out/ncu_f.log
