#!/bin/bash
# full GPU suite + default bench line + reference arm (round-end refresh)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/gpu_suite.txt
cat gpurun_out/gpu_suite.txt
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -1 gpurun_out/bench_final.json | cut -c1-400
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err
tail -1 gpurun_out/bench_ref_final.json | cut -c1-300
