#!/bin/bash
# EKS_MPK=force integration test + CA / matrix-powers regression
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "matrix_powers or ca_end_to_end" 2>&1 | tail -25 > gpurun_out/mpk_tests2.txt
cat gpurun_out/mpk_tests2.txt
