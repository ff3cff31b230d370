EKS_SPMM_PATH=grid timeout 900 python -m pytest tests -m gpu -x -q -k "spmm or cfg1 or basis or full_size or cfg2_full or cfg4_analog" 2>&1 | tail -3
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4,cfg5 --ts 8,16,32,64 --variants 2,6 2>&1 | grep -v "^#"
