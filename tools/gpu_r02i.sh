#!/bin/bash
# round-2 call I: evidence — fp64 peaks (incl. DMMA+DFMA), SpMM by=4/8 A/B, cfg4 solve profile,
# ncu launch list + full capture of the cfg5 sweep kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/full_solves.py --cfg cfg4 --profile --out gpurun_out/i_full.jsonl > gpurun_out/i_cfg4.log 2>&1; echo "cfg4 rc=$?" >> gpurun_out/i_rc.txt
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 8 > gpurun_out/i_sweep_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launches_cfg5.csv python tools/sweep_once.py --N 384 --t 16 --nblocks 8 > gpurun_out/i_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/i_rc.txt
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/i_sweep4_plain.txt 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_apply_tc|k_spmm_grid" -s 8 -c 5 -o gpurun_out/i_cfg5_full python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/i_ncu_full.log 2>&1
rc=$?; echo "full rc=$rc" >> gpurun_out/i_rc.txt
if [ $rc -ne 0 ]; then
  timeout 600 python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/i_sweep256_plain.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_apply_tc|k_spmm_grid" -s 8 -c 5 -o gpurun_out/i_cfg4size_full python tools/sweep_once.py --N 256 --t 16 --nblocks 4 > gpurun_out/i_ncu_full256.log 2>&1
  echo "full256 rc=$?" >> gpurun_out/i_rc.txt
fi
for T in 32 64; do
  SK=1; [ $T -eq 64 ] && SK=2
  timeout 600 python tools/spmm_once.py --N 384 --t $T > gpurun_out/i_spmm${T}_plain.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmm_grid|k_sweep" -s $SK -c $SK -o gpurun_out/i_spmm${T}_full python tools/spmm_once.py --N 384 --t $T > gpurun_out/i_ncu_spmm$T.log 2>&1
  echo "spmm$T rc=$?" >> gpurun_out/i_rc.txt
done
# export the captures here (the .ncu-rep files of 384^3 kernels exceed gpurun's 64 MiB copy-back)
for f in gpurun_out/*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"
  sz=$(stat -c %s "$f"); if [ "$sz" -gt 12000000 ]; then rm -f "$f"; fi
done
du -sh gpurun_out
exit 0
