#!/bin/bash
# round-2 call R: t=32 warp-owned-row kernels (k_upcoef_w<32>, k_apply_tc<32> WOWN): parity, cfg5 t=32 A/B, ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "basis_sweep or onesynch_end or large_t or cgs2_and_acholqr or graph_replay or cfg2_analog" > gpurun_out/r_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r_rc.txt
tail -2 gpurun_out/r_tests.log
for V in 1 0; do
  EKS_UPCOEF16=$V timeout 900 python bench.py --t 32 --s 8 --steps 2 --warmup 3 --no-cpu --no-e2e --no-spmm-block --extra , > gpurun_out/r_t32_$V.json 2> gpurun_out/r_t32_$V.err; echo "t32 V=$V rc=$?" >> gpurun_out/r_rc.txt
  python -c "
import json; d=json.loads(open('gpurun_out/r_t32_$V.json').read().splitlines()[-1])
print('t32 V=$V', round(d['value'],3), round(d['sweep']['frac_of_hbm'],3), d['clocks']['sm_mhz'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items() if k!='chol'})"
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --extra cfg2 > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?" >> gpurun_out/r_rc.txt
python -c "
import json; d=json.loads(open('gpurun_out/r_bench.json').read().splitlines()[-1])
print('t16 bench', d['value'], d['clocks'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items()}, d['extras'].get('cfg2',{}).get('outer_it_per_s'), d['e2e']['value'], {t: round(v['frac'],3) for t, v in d['spmm_block']['t'].items()})"
timeout 600 python tools/sweep_once.py --N 384 --t 32 --nblocks 4 > gpurun_out/r_sweep_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_upcoef_w|k_apply_tc" -s 2 -c 2 -o gpurun_out/r_t32 python tools/sweep_once.py --N 384 --t 32 --nblocks 4 > gpurun_out/r_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r_rc.txt
for f in gpurun_out/r_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/r_rc.txt
exit 0
