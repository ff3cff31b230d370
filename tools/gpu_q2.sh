timeout 600 python -m pytest tests -m gpu -x -q -k "not cfg2_analog_end_to_end and not cfg3_analog" > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4 --ts 8,16,32,64 > gpurun_out/micro.log 2>&1; cat gpurun_out/micro.log
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-200; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['time_share'], d['spmm_roofline']['avg_launch_us'])"
