for c in 1 4 16 64; do echo "chunk=$c"; EKS_SPMM_CHUNK=$c timeout 600 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4 --ts 8,16,32,64 --variants 1 2>&1 | grep -v "^#"; done
