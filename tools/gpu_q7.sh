timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg2_analog_end_to_end and not cfg3_analog" 2>&1 | tail -2
for p in 0 1; do EKS_PDL=$p timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_pdl$p.log 2>&1; echo "pdl=$p"; tail -1 gpurun_out/bench_pdl$p.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
