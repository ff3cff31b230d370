#!/bin/bash
# round-2 call U (final): full GPU suite, smoke, default bench line, reference arm, ncu launch list of a
# short headline run, --set full capture of the headline kernels (summaries + DRAM traffic into profiles/)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/u_suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/u_rc.txt
tail -3 gpurun_out/u_suite.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/u_rc.txt
tail -1 gpurun_out/u_smoke.log
timeout 1500 python bench.py > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err; echo "bench rc=$?" >> gpurun_out/u_rc.txt
tail -1 gpurun_out/u_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/u_ref.json 2> gpurun_out/u_ref.err; echo "ref rc=$?" >> gpurun_out/u_rc.txt
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --extra ,"
timeout 600 $SHORT > gpurun_out/u_short_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/u_launches_cfg5.csv $SHORT > gpurun_out/u_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/u_rc.txt
timeout 600 python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/u_sweep_plain.txt 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_upcoef_w|k_sweep|k_apply_tc|k_spmm_grid" -s 8 -c 4 -o gpurun_out/u_cfg5_full python tools/sweep_once.py --N 384 --t 16 --nblocks 4 > gpurun_out/u_ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/u_rc.txt
for f in gpurun_out/u_*.ncu-rep; do
  [ -f "$f" ] || continue
  b="${f%.ncu-rep}"
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
  ncu -i "$f" --page source --csv --print-source sass > "$b.source.csv" 2>/dev/null
  gzip -f "$b.source.csv"; rm -f "$f"
done
cat gpurun_out/u_rc.txt
exit 0
