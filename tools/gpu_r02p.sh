#!/bin/bash
# round-2 call P: t=8 Y-scratch fix (5 stages again) — SpMM micro t=8/16/32, SpMM parity, and the
# cfg5 sweep over t in {8,16,32} x s in {2,4,8} (BASELINE configs[4]) with the current kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/spmm_micro.py --ops cfg5 --ts 8,16,32 --variants 7 --reps 10 > gpurun_out/p_micro.txt 2>&1; echo "micro rc=$?" >> gpurun_out/p_rc.txt
cat gpurun_out/p_micro.txt | grep cfg5
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or basis_sweep_parity" > gpurun_out/p_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/p_rc.txt
tail -2 gpurun_out/p_tests.log
for T in 8 16 32; do for S in 2 4 8; do
  timeout 900 python bench.py --t $T --s $S --steps 2 --warmup 3 --no-cpu --no-e2e --no-spmm-block --extra , > gpurun_out/p_cfg5_t${T}_s${S}.json 2> gpurun_out/p_cfg5_t${T}_s${S}.err
  echo "t$T s$S rc=$?" >> gpurun_out/p_rc.txt
  python -c "
import json; d=json.loads(open('gpurun_out/p_cfg5_t${T}_s${S}.json').read().splitlines()[-1])
print('t=$T s=$S', round(d['value'],3), round(d['sweep']['frac_of_hbm'],3), d['clocks']['sm_mhz'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items() if k!='chol'})"
done; done
cat gpurun_out/p_rc.txt
exit 0
