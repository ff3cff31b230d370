#!/bin/bash
# Round-end profile refresh of the default bench command (B200_PROFILING.md recipe): the plain run
# first, then the ncu launch list of the same command, then one --set full capture of the top
# kernels of a short solve (read back here with tools/ncu_summary.py / tools/launch_summary.py).
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-spmm-block"
$CMD > gpurun_out/profile_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01.csv \
    $CMD > gpurun_out/ncu_launches.log 2>&1
SHORT="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-spmm-block --max-outer 20"
ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_spmm_grid|k_apply_tc|k_chol_fast" \
    -s 60 -c 6 -o gpurun_out/prof_full $SHORT > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
