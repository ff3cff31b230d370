#!/bin/bash
# round-2 call J: pair-major stencil values, ZT apply, full unroll restored: tests, micro, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or basis_sweep or path_size or cfg2_analog or cfg1_end or graph_replay or ca_end" > gpurun_out/j_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/j_rc.txt
timeout 900 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32,64 --variants 7 --reps 10 > gpurun_out/j_micro.txt 2>&1
EKS_GRID_PATCH=0 timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16 --variants 7 --reps 10 > gpurun_out/j_micro_p0.txt 2>&1
EKS_GRID_BY=8 timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16,32 --variants 7 --reps 10 > gpurun_out/j_micro_by8.txt 2>&1
timeout 1200 python bench.py > gpurun_out/j_bench.json 2> gpurun_out/j_bench.err; echo "bench rc=$?" >> gpurun_out/j_rc.txt
exit 0
