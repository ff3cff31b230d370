#!/bin/bash
# plane-block height sweep of the plane-marching SpMM-block kernel (cfg5 and cfg4 operators)
for by in 4 8 16; do
  echo "== by=$by"
  EKS_GRID_BY=$by timeout 600 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32 --variants 2 --reps 10 2>&1 | grep -v "^#"
done
