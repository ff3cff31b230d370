for p in 0 1; do echo "probe=$p"; EKS_SEG_PROBE=$p timeout 600 python tools/spmm_micro.py --ops cfg2,cfg4 --ts 8,16,32,64 --variants 1 2>&1 | grep -v "^#"; done > gpurun_out/probe2.log 2>&1
