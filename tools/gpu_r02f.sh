#!/bin/bash
# round-2 call F: variants on cfg2 (precond IC(0) with column-group trsv, CA SRE-CG s=2 with plane-marching
# powers), cfg3 full size (store-Q-only), ncu evidence of the cfg5 kernels (launch list + full capture)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "precond or trsv or ca_" > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f_rc.txt
timeout 600 python bench.py --workload cfg2 --precond 64 --no-spmm-block --no-e2e > gpurun_out/f_bench_precond.json 2> gpurun_out/f_bench_precond.err; echo "precond rc=$?" >> gpurun_out/f_rc.txt
timeout 600 python bench.py --workload cfg2 --method ca-sre-cg --s 2 --no-spmm-block --no-e2e > gpurun_out/f_bench_ca.json 2> gpurun_out/f_bench_ca.err; echo "ca rc=$?" >> gpurun_out/f_rc.txt
timeout 600 python bench.py --workload cfg2 --no-spmm-block > gpurun_out/f_bench_cfg2.json 2> gpurun_out/f_bench_cfg2.err; echo "cfg2 rc=$?" >> gpurun_out/f_rc.txt
timeout 1500 python tools/full_solves.py --cfg cfg3 --max-outer 2000 --profile --out gpurun_out/f_full.jsonl > gpurun_out/f_cfg3.log 2>&1; echo "cfg3 rc=$?" >> gpurun_out/f_rc.txt
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 8 > gpurun_out/f_sweep_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_cfg5.csv python tools/sweep_once.py --N 384 --t 16 --nblocks 8 > gpurun_out/f_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/f_rc.txt
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/f_sweep4_plain.txt 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_apply_tc|k_spmm_grid" -s 8 -c 5 -o gpurun_out/f_cfg5_full python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/f_ncu_full.log 2>&1
rc=$?; echo "full rc=$rc" >> gpurun_out/f_rc.txt
if [ $rc -ne 0 ]; then
  timeout 600 python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/f_sweep256_plain.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_apply_tc|k_spmm_grid" -s 8 -c 5 -o gpurun_out/f_cfg4size_full python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/f_ncu_full256.log 2>&1
  echo "full256 rc=$?" >> gpurun_out/f_rc.txt
fi
exit 0
