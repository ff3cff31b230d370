nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/gpu_tests.log 2>&1; tail -12 gpurun_out/gpu_tests.log
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-2000
