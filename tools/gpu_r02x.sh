#!/bin/bash
# device-resident loop (use_graph = 2): parity tests, cfg1/cfg2 timing of modes 0/1/2, default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "device_loop or graph_replay" 2>&1 | tail -25 > gpurun_out/dloop_tests.txt
cat gpurun_out/dloop_tests.txt
timeout 600 python tools/graph_timing.py > gpurun_out/graph_timing.txt 2>&1
cat gpurun_out/graph_timing.txt
timeout 900 python bench.py > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
tail -1 gpurun_out/bench_x.json | cut -c1-600
