# full ncu capture of selected kernels of one cfg2 solve (capped at 20 outer iterations)
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on \
  --kernel-name-base function -k regex:"${NCU_K:-k_spmm_gram|k_apply_tc}" -s ${NCU_S:-200} -c ${NCU_C:-2} \
  -o gpurun_out/${NCU_O:-prof} $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
