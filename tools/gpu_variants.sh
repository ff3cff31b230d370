#!/bin/bash
# bench lines of the §8(f) variants on cfg2 (s=3, t=16 unless stated)
mkdir -p gpurun_out
run() {
  name=$1; shift
  timeout 400 python bench.py --steps 3 --warmup 3 --no-spmm-block --cpu-iters 1 "$@" > gpurun_out/bench_$name.json 2> gpurun_out/bench_$name.err
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{name}.json").read().strip().splitlines()[-1])
    print(name, round(d["value"], 1), round(d["ms_per_step"], 1), d["solve"]["outer_iters"], round(d["e2e"]["value"], 1),
          d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), {k: round(v, 3) for k, v in d["time_share"].items() if v > 0.005})
except Exception as e:
    print(name, "FAILED", open(f"gpurun_out/bench_{name}.err").read()[-400:])
PY
}
for v in $VARIANTS; do
  case $v in
    ca2) run ca2 --method ca-sre-cg --s 2 ;;
    restr) run restr --restructured ;;
    pre) run pre --ortho pre-cholqr ;;
    prec) run prec --precond 64 ;;
    chol) run chol --precond 64 --precond-kind chol --no-cpu --no-e2e --max-outer 4 --steps 2 ;;
  esac
done
