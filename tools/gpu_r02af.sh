#!/bin/bash
# final: smoke(), full GPU suite, default bench line, ncu launch list (final code)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3 > gpurun_out/smoke.txt
cat gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -1 gpurun_out/bench_final.json | cut -c1-300
timeout 2400 python -m pytest tests -m gpu -q --durations=8 2>&1 | tail -24 > gpurun_out/gpu_suite_full.txt
tail -3 gpurun_out/gpu_suite_full.txt
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-spmm-block --extra ,"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv \
    $CMD > gpurun_out/ncu_launches.log 2>&1
tail -1 gpurun_out/ncu_launches.log | cut -c1-200
