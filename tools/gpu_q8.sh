timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['spmm_block']), d['roofline'])"
timeout 900 python bench.py --workload cfg5 --steps 2 --warmup 1 > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | cut -c1-1500
