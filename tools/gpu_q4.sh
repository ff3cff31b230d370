timeout 600 python -m pytest tests -m gpu -x -q -k "spmm or cgs2 or basis or cfg1" > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4,cfg5 --ts 8,16,32,64 --variants 0,4,1,3 > gpurun_out/micro.log 2>&1; cat gpurun_out/micro.log
