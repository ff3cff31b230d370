#!/bin/bash
# round-2 call G: lazy-basis fix, swizzled-TMA t=16 SpMM: tests, micro, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or graph_replay or path_size or cfg2_full_size or cfg4_analog or cfg2_analog or preconditioned_end or large_t or solve_prefix or basis_sweep" > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g_rc.txt
timeout 600 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 16 --variants 2 --reps 10 > gpurun_out/g_micro.txt 2>&1
EKS_GRID_PATCH=0 timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16 --variants 2 --reps 10 > gpurun_out/g_micro_p0.txt 2>&1
timeout 1200 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?" >> gpurun_out/g_rc.txt
exit 0
