free -g | head -2
timeout 900 python tools/spmm_micro.py --ops ${OPS:-cfg2,cfg3,cfg4} --ts ${TS:-8,16,32,64} > gpurun_out/micro.log 2>&1; cat gpurun_out/micro.log
