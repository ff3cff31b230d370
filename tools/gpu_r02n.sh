#!/bin/bash
# round-2 call N: one-synch GPU tests + per-warp C1 apply (WOWN): parity subset, short cfg5 bench, ncu of the apply
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "onesynch or cgs2_and_acholqr or cfg2_analog or path_size or basis_sweep or graph_replay or cfg1_end_to_end or determinism" > gpurun_out/n_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/n_rc.txt
tail -3 gpurun_out/n_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --extra cfg2 > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench rc=$?" >> gpurun_out/n_rc.txt
python -c "
import json; d=json.loads(open('gpurun_out/n_bench.json').read().splitlines()[-1])
print(d['value'], d['clocks'], {k:(round(v['avg_launch_us'],1), round(v['frac'],3)) for k,v in d['per_class'].items()}, d['extras'].get('cfg2',{}).get('outer_it_per_s'))"
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/n_sweep4_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply_tc" -s 2 -c 1 -o gpurun_out/n_apply_full python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/n_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/n_rc.txt
for f in gpurun_out/n_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/n_rc.txt
exit 0
