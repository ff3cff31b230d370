#!/bin/bash
python -m pytest tests/test_gpu_parity.py -m gpu -k "precond" -q -x 2>&1 | tail -2
VARIANTS="prec" bash tools/gpu_variants.sh
EKS_TRSV_WARP=0 VARIANTS="prec" bash tools/gpu_variants.sh
