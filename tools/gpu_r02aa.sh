#!/bin/bash
# setup with the CSR upload under the validation: setup/error-path tests, setup timing, default bench,
# reference arm, ncu launch list of the default bench command
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bad_matrix or errors or spmm_bitwise or matrix_powers or cfg4 or cgs2" 2>&1 | tail -6 > gpurun_out/setup_tests.txt
cat gpurun_out/setup_tests.txt
timeout 600 python tools/spmm_micro.py --ops cfg4 --ts 64 --variants 7 --reps 10 > gpurun_out/spmm_micro_t64.txt 2>&1
tail -2 gpurun_out/spmm_micro_t64.txt
timeout 600 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1
tail -4 gpurun_out/e2e_breakdown.txt
timeout 600 python tools/setup_timing.py > gpurun_out/setup_timing.txt 2>&1
tail -12 gpurun_out/setup_timing.txt
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -1 gpurun_out/bench_final.json | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
tail -1 gpurun_out/bench_ref_final.json | cut -c1-300
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-spmm-block --extra ,"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv \
    $CMD > gpurun_out/ncu_launches.log 2>&1
tail -2 gpurun_out/ncu_launches.log | cut -c1-200
