#!/bin/bash
# round-2 call C: ncu of the grid SpMM (patch vs per-row) and of the sweep kernels; new tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for P in 1 0; do
  EKS_GRID_PATCH=$P timeout 300 python tools/spmm_micro.py --ops cfg4 --ts 16,32 --variants 2 --reps 10 > gpurun_out/c_micro_p$P.txt 2>&1
done
timeout 300 python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/c_sweep_plain.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "store_q_only or spmm_bitwise or basis_sweep_parity or cfg2_analog or graph_replay" > gpurun_out/c_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/c_rc.txt
for P in 1 0; do
  EKS_GRID_PATCH=$P timeout 300 python tools/spmm_micro.py --ops cfg4 --ts 16 --variants 2 --reps 1 > gpurun_out/c_plain_p$P.txt 2>&1 && \
  EKS_GRID_PATCH=$P timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm_grid -s 1 -c 1 -o gpurun_out/c_grid16_p$P python tools/spmm_micro.py --ops cfg4 --ts 16 --variants 2 --reps 1 > gpurun_out/c_ncu_p$P.log 2>&1
  echo "ncu$P rc=$?" >> gpurun_out/c_rc.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_apply_tc" -s 6 -c 4 -o gpurun_out/c_sweep16 python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/c_ncu_sweep.log 2>&1; echo "ncusw rc=$?" >> gpurun_out/c_rc.txt
exit 0
