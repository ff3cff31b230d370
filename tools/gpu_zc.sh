#!/bin/bash
for zc in 0 2 3 4 6 16; do
  EKS_GRID_ZC=$zc timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-spmm-block > gpurun_out/zc_$zc.json 2>/dev/null
  python - $zc <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/zc_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("zc", sys.argv[1], round(d["value"],1), "spmm us/launch", round(d["spmm_roofline"]["avg_launch_us"],2), "frac", round(d["spmm_roofline"]["frac"],3))
PY
done
