#!/bin/bash
# device-resident loop (use_graph = 2): parity tests, cfg1/cfg2 timing of modes 0/1/2
mkdir -p gpurun_out
python -c "from paper_1804_10629_b200 import build as b; b.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "device_loop or graph_replay" 2>&1 | tail -5 > gpurun_out/dloop_tests.txt
cat gpurun_out/dloop_tests.txt
timeout 600 python tools/graph_timing.py > gpurun_out/graph_timing.txt 2>&1
cat gpurun_out/graph_timing.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=40 2>&1 | tail -60 > gpurun_out/gpu_suite_full.txt
tail -3 gpurun_out/gpu_suite_full.txt
