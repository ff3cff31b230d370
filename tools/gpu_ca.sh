#!/bin/bash
# CA parity tests + CA bench line on cfg2 (s=2; s=3 breaks down on both sides)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -k "ca_" -q -x 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 3 --no-spmm-block --method ca-sre-cg --s 2 --cpu-iters 2 > gpurun_out/bench_ca.json 2> gpurun_out/bench_ca.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_ca.json").read().strip().splitlines()[-1])
print(round(d["value"],1), d["ms_per_step"], d["solve"]["outer_iters"], d["e2e"]["value"], d["cpu_baseline"]["value"])
print({k:round(v,3) for k,v in d.get("time_share",{}).items()}, d["roofline"]["kernel"], round(d["roofline"]["frac"],3))
PY
