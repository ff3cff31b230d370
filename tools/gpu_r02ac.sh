#!/bin/bash
# final evidence: ncu --set full of the t=64 SpMM-block step (k_spmm_grid<64> Gram-free + k_gram_w<64> with FMA X^T v)
# at 384^3; refreshed CA / preconditioned cfg2 bench lines
mkdir -p gpurun_out
timeout 600 python tools/spmm_once.py --N 384 --t 64 > gpurun_out/ac_spmm64_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_w|k_spmm_grid" -s 2 -c 2 -o gpurun_out/ac_spmm64 python tools/spmm_once.py --N 384 --t 64 > gpurun_out/ac_ncu.log 2>&1
echo "ncu rc=$?"
for f in gpurun_out/ac_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  rm -f "$f"
done
cat gpurun_out/ac_spmm64_plain.txt | tail -1
timeout 600 python bench.py --workload cfg2 --method ca-sre-cg --s 2 --no-cpu > gpurun_out/ac_bench_ca.json 2> gpurun_out/ac_bench_ca.err
tail -1 gpurun_out/ac_bench_ca.json | cut -c1-200
timeout 600 python bench.py --workload cfg2 --precond 64 --no-cpu > gpurun_out/ac_bench_prec.json 2> gpurun_out/ac_bench_prec.err
tail -1 gpurun_out/ac_bench_prec.json | cut -c1-200
