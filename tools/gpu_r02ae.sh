#!/bin/bash
# X^T r on the FMA pipe in k_spmm_grid: parity subset + SpMM-block micro at 384^3
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "spmm_bitwise or cgs2_and_acholqr or end_to_end_sre or full_size_spmm or cfg2_prefix or smoke or graph_replay or device_loop" 2>&1 | tail -6 > gpurun_out/ae_tests.txt
cat gpurun_out/ae_tests.txt
timeout 900 python tools/spmm_micro.py --ops cfg5 --ts 8,16,32 --variants 7 --reps 10 > gpurun_out/ae_micro.txt 2>&1
grep cfg5 gpurun_out/ae_micro.txt
