#!/bin/bash
# round-2 call K: register-gathered Gram fragments in the t=16 patch SpMM: tests, micro, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32,64 --variants 7 --reps 10 > gpurun_out/k_micro.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or basis_sweep or path_size or cfg2_analog or graph_replay" > gpurun_out/k_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k_rc.txt
timeout 1200 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; echo "bench rc=$?" >> gpurun_out/k_rc.txt
exit 0
