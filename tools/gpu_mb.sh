for mb in 0 4 6 8; do echo "minb=$mb"; EKS_ELL_MINB=$mb timeout 600 python tools/spmm_micro.py --ops cfg3,cfg4 --ts 16 --variants 1 2>&1 | grep -v "^#"; done > gpurun_out/mb.log 2>&1
