# tests + short bench + launch list
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/gpu_tests.log 2>&1; tail -4 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
