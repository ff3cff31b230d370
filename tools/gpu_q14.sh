timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['spmm_roofline']['frac'], json.dumps(d['spmm_block']['t']))"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-spmm-block --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv | head -8
