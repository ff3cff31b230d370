./tools/chol_probe
timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg2_analog_end_to_end and not cfg3_analog" 2>&1 | tail -3
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['time_share'], d['spmm_roofline']['avg_launch_us'])"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv
