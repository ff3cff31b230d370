#!/bin/bash
# round-2 call O: k_upcoef16 (swizzled, warp-owned rows) + device-side stencil values at setup:
# parity subset, bench A/B (EKS_UPCOEF16=0/1), ncu of the new kernel
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "onesynch or cfg2_analog or path_size or basis_sweep or graph_replay or full_size or spmm_bitwise or determinism" > gpurun_out/o_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/o_rc.txt
tail -3 gpurun_out/o_tests.log
for V in 1 0; do
  EKS_UPCOEF16=$V timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --extra cfg2 > gpurun_out/o_bench$V.json 2> gpurun_out/o_bench$V.err; echo "bench$V rc=$?" >> gpurun_out/o_rc.txt
  python -c "
import json; d=json.loads(open('gpurun_out/o_bench$V.json').read().splitlines()[-1])
print('V=$V', d['value'], d['clocks'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items()}, d['extras'].get('cfg2',{}).get('outer_it_per_s'), d['e2e'])"
done
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/o_sweep4_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_upcoef16|k_apply_tc" -s 2 -c 2 -o gpurun_out/o_full python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/o_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/o_rc.txt
for f in gpurun_out/o_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/o_rc.txt
exit 0
