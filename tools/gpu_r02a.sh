#!/bin/bash
# round-2 first GPU call: smoke, new parity tests, full-size cfg4/cfg3 solves
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 600 python __graft_entry__.py smoke > gpurun_out/a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/a_rc.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "path_size_prefix or graph_replay or trsv_ring or full_size_spmm_gram or pre_cholqr_restructured_end or preconditioned_end" > gpurun_out/a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/a_rc.txt
timeout 900 python tools/full_solves.py --cfg cfg4 --max-outer 3000 --out gpurun_out/a_full.jsonl > gpurun_out/a_cfg4.log 2>&1; echo "cfg4 rc=$?" >> gpurun_out/a_rc.txt
timeout 900 python tools/full_solves.py --cfg cfg3 --max-outer 400 --out gpurun_out/a_full.jsonl > gpurun_out/a_cfg3.log 2>&1; echo "cfg3 rc=$?" >> gpurun_out/a_rc.txt
exit 0
