#!/bin/bash
# round-2 call Q: FRAG-layout t=16 plane-marching SpMM (EKS_GRID_PV=3): micro A/B, parity, bench, ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for V in 0 3; do EKS_GRID_PV=$V timeout 600 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 16 --variants 7 --reps 10 > gpurun_out/q_micro_pv$V.txt 2>&1; grep cfg gpurun_out/q_micro_pv$V.txt | sed "s/^/PV=$V /"; done
EKS_GRID_PV=3 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or basis_sweep or cfg3_analog or cfg4_analog" > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/q_rc.txt
tail -2 gpurun_out/q_tests.log
EKS_GRID_PV=3 timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra , > gpurun_out/q_bench3.json 2> gpurun_out/q_bench3.err; echo "bench rc=$?" >> gpurun_out/q_rc.txt
python -c "
import json; d=json.loads(open('gpurun_out/q_bench3.json').read().splitlines()[-1])
print('PV=3 bench', d['value'], d['clocks'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items()}, {t: round(v['frac'],3) for t, v in d['spmm_block']['t'].items()})"
EKS_GRID_PV=3 timeout 600 python tools/spmm_once.py --N 384 --t 16 > gpurun_out/q_spmm_plain.txt 2>&1 && \
EKS_GRID_PV=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_grid" -s 1 -c 1 -o gpurun_out/q_spmm16 python tools/spmm_once.py --N 384 --t 16 > gpurun_out/q_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/q_rc.txt
for f in gpurun_out/q_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/q_rc.txt
exit 0
