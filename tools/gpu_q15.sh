timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/debug_t64.py 64 2 2>&1 | tail -2
OP=cfg5 python tools/debug_t64.py 16 2 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['spmm_roofline']['frac'], json.dumps(d['spmm_block']['t']))"
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg3,cfg4,cfg5 --ts 8,16,32,64 --variants 0,4,2 > gpurun_out/micro.log 2>&1; cat gpurun_out/micro.log
