#!/bin/bash
# round-2 call D: 1x4-patch SpMM A/B, full GPU suite, default bench (cfg5 headline), reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for P in 1 0; do
  EKS_GRID_PATCH=$P timeout 600 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 16,32 --variants 2 --reps 10 > gpurun_out/d_micro_p$P.txt 2>&1
done
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/d_rc.txt
timeout 1200 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err; echo "bench rc=$?" >> gpurun_out/d_rc.txt
timeout 900 python bench.py --impl reference > gpurun_out/d_ref.json 2> gpurun_out/d_ref.err; echo "ref rc=$?" >> gpurun_out/d_rc.txt
exit 0
