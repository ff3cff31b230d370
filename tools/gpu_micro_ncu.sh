CMD="python tools/spmm_micro.py --ops ${OPS:-cfg4} --ts ${TS:-16} --variants ${VARS:-0,1} --reps 2"
$CMD > gpurun_out/micro_plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base function -k regex:"k_spmm" -s ${NCU_S:-0} -c ${NCU_C:-6} -o gpurun_out/${NCU_O:-micro} $CMD > gpurun_out/micro_ncu.log 2>&1
tail -3 gpurun_out/micro_ncu.log; cat gpurun_out/micro_plain.log
