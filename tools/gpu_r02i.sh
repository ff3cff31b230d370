#!/bin/bash
# round-2 call I: evidence — fp64 peaks (incl. DMMA+DFMA), SpMM by=4/8 A/B, cfg4 solve profile,
# ncu launch list + full capture of the cfg5 sweep kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
./tools/fp64_peaks > gpurun_out/i_fp64.txt 2>&1
timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16,32 --variants 2 --reps 10 > gpurun_out/i_micro_by4.txt 2>&1
EKS_GRID_BY=8 timeout 600 python tools/spmm_micro.py --ops cfg5 --ts 16,32 --variants 2 --reps 10 > gpurun_out/i_micro_by8.txt 2>&1
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
exit 0
