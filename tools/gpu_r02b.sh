#!/bin/bash
# round-2 call B: fp64 pipe test, patch SpMM A/B + parity, cfg3 analog iteration counts
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
free -g > gpurun_out/b_host.txt; nproc >> gpurun_out/b_host.txt
./tools/fp64_peaks > gpurun_out/b_fp64.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm_gram or basis_sweep_parity or cfg2_analog or graph_replay_bitwise or path_size" > gpurun_out/b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/b_rc.txt
for P in 1 0; do
  EKS_GRID_PATCH=$P timeout 600 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 16,32 --variants 2 > gpurun_out/b_micro_patch$P.txt 2>&1; echo "micro$P rc=$?" >> gpurun_out/b_rc.txt
done
for N in 32 64; do
  timeout 600 python tools/full_solves.py --cfg cfg3 --N $N --max-outer 2000 --out gpurun_out/b_full.jsonl > gpurun_out/b_cfg3_$N.log 2>&1; echo "cfg3_$N rc=$?" >> gpurun_out/b_rc.txt
done
exit 0
