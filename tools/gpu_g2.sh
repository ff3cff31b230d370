# parity tests (fast subset first), short bench, launch list
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/gpu_tests.log 2>&1; tail -15 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log | cut -c1-2500
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; tail -2 gpurun_out/ncu.log
