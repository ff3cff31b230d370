#!/bin/bash
# round-2 call L: t=16 patch variants A/B in one box (scratch / shuffles / per-row), then the evidence
# captures (call I script)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for V in 0 2; do EKS_GRID_PV=$V timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16 --variants 7 --reps 10 > gpurun_out/l_micro_pv$V.txt 2>&1; done
EKS_GRID_PATCH=0 timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16 --variants 7 --reps 10 > gpurun_out/l_micro_p0.txt 2>&1
bash tools/gpu_r02i.sh
exit 0
