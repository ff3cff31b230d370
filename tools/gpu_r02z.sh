#!/bin/bash
# full GPU suite with durations (round-2 refresh)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -45 > gpurun_out/gpu_suite_full.txt
tail -3 gpurun_out/gpu_suite_full.txt
