#!/bin/bash
for pth in grid ell csr; do
  EKS_SPMM_PATH=$pth timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-spmm-block > gpurun_out/path_$pth.json 2>/dev/null
  python - $pth <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/path_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("path", sys.argv[1], round(d["value"],1), "spmm us/launch", round(d["spmm_roofline"]["avg_launch_us"],2), "frac", round(d["spmm_roofline"]["frac"],3))
PY
done
