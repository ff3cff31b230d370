#!/bin/bash
# round-2 call H: full GPU suite, SpMM micro (t=16 patch, t=64 Gram-free patch), bench, cfg2 variants, cfg3 full size
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32,64 --variants 2,7 --reps 10 > gpurun_out/h_micro.txt 2>&1
timeout 1200 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$?" >> gpurun_out/h_rc.txt
timeout 600 python bench.py --workload cfg2 --precond 64 --no-spmm-block --no-e2e > gpurun_out/h_bench_precond.json 2> gpurun_out/h_bench_precond.err; echo "precond rc=$?" >> gpurun_out/h_rc.txt
timeout 600 python bench.py --workload cfg2 --method ca-sre-cg --s 2 --no-spmm-block --no-e2e > gpurun_out/h_bench_ca.json 2> gpurun_out/h_bench_ca.err; echo "ca rc=$?" >> gpurun_out/h_rc.txt
timeout 600 python bench.py --workload cfg2 --no-spmm-block > gpurun_out/h_bench_cfg2.json 2> gpurun_out/h_bench_cfg2.err; echo "cfg2 rc=$?" >> gpurun_out/h_rc.txt
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/h_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/h_rc.txt
timeout 1500 python tools/full_solves.py --cfg cfg3 --max-outer 2000 --out gpurun_out/h_full.jsonl > gpurun_out/h_cfg3.log 2>&1; echo "cfg3 rc=$?" >> gpurun_out/h_rc.txt
exit 0
