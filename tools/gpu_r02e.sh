#!/bin/bash
# round-2 call E: lazy basis + t=64 split Gram + parallel setup: micro, full GPU suite, bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32,64 --variants 2,7 --reps 10 > gpurun_out/e_micro.txt 2>&1
EKS_GRAM64=fused timeout 600 python tools/spmm_micro.py --ops cfg4 --ts 64 --variants 7 --reps 5 > gpurun_out/e_micro_fused64.txt 2>&1
timeout 1200 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo "bench rc=$?" >> gpurun_out/e_rc.txt
EKS_LAZY_W=0 timeout 1200 python bench.py --no-e2e --no-cpu --no-spmm-block --extra "" > gpurun_out/e_bench_eager.json 2> gpurun_out/e_bench_eager.err; echo "bench_eager rc=$?" >> gpurun_out/e_rc.txt
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/e_rc.txt
exit 0
