for t in 16 32; do
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"k_spmm_grid" -c 1 -o gpurun_out/grid_t$t python tools/spmm_micro.py --ops cfg4 --ts $t --variants 2 --reps 1 > gpurun_out/ncu_g$t.log 2>&1
done
