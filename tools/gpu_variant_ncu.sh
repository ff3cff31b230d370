#!/bin/bash
# smoke + ncu launch lists of the §8(f) variants on cfg2 (plain runs first, then under ncu)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-spmm-block"
$B --method ca-sre-cg --s 2 --max-outer 6 > /dev/null 2>&1 && echo ca-ok
$B --precond 64 --max-outer 6 > /dev/null 2>&1 && echo prec-ok
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_ca_r01.csv $B --method ca-sre-cg --s 2 --max-outer 6 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_precond_r01.csv $B --precond 64 --max-outer 6 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_trsv_ring" -s 4 -c 1 -o gpurun_out/ncu_trsv_r01 $B --precond 64 --max-outer 6 > /dev/null 2>&1
ls -la gpurun_out | tail -5
