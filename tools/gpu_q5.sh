timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
EKS_SPMM_PATH=ell timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['time_share'], d['spmm_roofline']['avg_launch_us'])"
CMD="python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --max-outer 20"
EKS_SPMM_PATH=ell $CMD > gpurun_out/plain.log 2>&1 && EKS_SPMM_PATH=ell timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 300 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1; python tools/launch_summary.py gpurun_out/launches.csv
