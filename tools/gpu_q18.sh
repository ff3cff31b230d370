timeout 900 python -m pytest tests -m gpu -x -q -k "spmm or cfg4_analog or basis or full_size or cgs2" 2>&1 | tail -2
timeout 900 python tools/spmm_micro.py --ops cfg2,cfg4,cfg5 --ts 32,64 --variants 2,6 2>&1 | grep -v "^#"
timeout 900 python bench.py --workload cfg4 --steps 1 --warmup 1 --max-outer 4 --no-cpu --no-e2e --no-spmm-block > gpurun_out/bench_cfg4.json 2>&1; tail -1 gpurun_out/bench_cfg4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['spmm_roofline']['frac'], d['time_share'])"
