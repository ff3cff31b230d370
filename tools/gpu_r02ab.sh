#!/bin/bash
# final: smoke() + full GPU suite with the final code
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -3 > gpurun_out/smoke.txt
cat gpurun_out/smoke.txt
timeout 2700 python -m pytest tests -m gpu -q --durations=12 2>&1 | tail -30 > gpurun_out/gpu_suite_full.txt
tail -3 gpurun_out/gpu_suite_full.txt
