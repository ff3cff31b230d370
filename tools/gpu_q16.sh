timeout 900 python -m pytest tests -m gpu -x -q -k "spmm or cfg4_analog or basis or full_size_spmm" 2>&1 | tail -2
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg4,cfg5 --ts 8,16,32,64 --variants 2,6 2>&1 | grep -v "^#"
