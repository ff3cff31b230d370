#!/bin/bash
# round-2 call S: padded X scratch for the SpMM Gram fragments (t=16 patch, t=32 per-row): micro, parity, bench, ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/spmm_micro.py --ops cfg5,cfg4 --ts 8,16,32 --variants 7 --reps 10 > gpurun_out/s_micro.txt 2>&1; echo "micro rc=$?" >> gpurun_out/s_rc.txt
grep cfg gpurun_out/s_micro.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "spmm_bitwise or full_size_spmm or basis_sweep or path_size or cfg3_analog or large_t or onesynch_path" > gpurun_out/s_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s_rc.txt
tail -2 gpurun_out/s_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --extra cfg2 > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err; echo "bench rc=$?" >> gpurun_out/s_rc.txt
python -c "
import json; d=json.loads(open('gpurun_out/s_bench.json').read().splitlines()[-1])
print('t16 bench', d['value'], d['clocks'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items()}, d['extras'].get('cfg2',{}).get('outer_it_per_s'), d['e2e']['value'], {t: round(v['frac'],3) for t, v in d['spmm_block']['t'].items()})"
for T in 16 32; do
timeout 600 python tools/spmm_once.py --N 384 --t $T > gpurun_out/s_spmm${T}_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_grid" -s 1 -c 1 -o gpurun_out/s_spmm$T python tools/spmm_once.py --N 384 --t $T > gpurun_out/s_ncu$T.log 2>&1
echo "ncu$T rc=$?" >> gpurun_out/s_rc.txt
done
for f in gpurun_out/s_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/s_rc.txt
exit 0
