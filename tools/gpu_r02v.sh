#!/bin/bash
# session re-entry check: smoke, full GPU suite, default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
tail -2 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/gpu_suite.txt
cat gpurun_out/gpu_suite.txt
python bench.py > gpurun_out/bench_v.json 2> gpurun_out/bench_v.err
tail -1 gpurun_out/bench_v.json | cut -c1-600
