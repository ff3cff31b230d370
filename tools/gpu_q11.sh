timeout 600 python -m pytest tests -m gpu -x -q -k "spmm" 2>&1 | tail -2
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4,cfg5 --ts 8,16,32 --variants 2 2>&1 | grep -v "^#"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"k_spmm_gram_ell" -c 1 python tools/spmm_micro.py --ops cfg5 --ts 16 --variants 2 --reps 1 2>&1 | grep -E "dram__|gpu__time"
