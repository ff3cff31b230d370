#!/bin/bash
# round-2 call T: warp-owned-row t=64 Gram sweep (k_gram_w<64>, EKS_GRAMW A/B): micro, parity, cfg4 solve, ncu
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for V in 1 0; do EKS_GRAMW=$V timeout 900 python tools/spmm_micro.py --ops cfg4,cfg5 --ts 64 --variants 7 --reps 5 > gpurun_out/t_micro$V.txt 2>&1; grep cfg gpurun_out/t_micro$V.txt | sed "s/^/GRAMW=$V /"; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "full_size_spmm or path_size or cfg4_analog or spmm_bitwise or cgs2_and_acholqr" > gpurun_out/t_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_rc.txt
tail -2 gpurun_out/t_tests.log
timeout 1200 python tools/full_solves.py --cfg cfg4 --profile --out gpurun_out/t_full.jsonl > gpurun_out/t_cfg4.log 2>&1; echo "cfg4 rc=$?" >> gpurun_out/t_rc.txt
python -c "
import json; d=json.loads(open('gpurun_out/t_full.jsonl').read().splitlines()[-1])
print('cfg4', d['status'], d['outer_iters'], d['outer_it_per_s'], d['true_relres'], {k: round(v,1) for k,v in d['profile_ms'].items() if v > 1})"
timeout 600 python tools/spmm_once.py --N 384 --t 64 > gpurun_out/t_spmm64_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_w|k_spmm_grid" -s 2 -c 2 -o gpurun_out/t_spmm64 python tools/spmm_once.py --N 384 --t 64 > gpurun_out/t_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/t_rc.txt
for f in gpurun_out/t_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/t_rc.txt
exit 0
