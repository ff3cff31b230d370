#!/bin/bash
# round-2 call M (re-entry): full GPU suite on HEAD, default bench line (cfg5 headline + extras),
# reference arm, ncu launch list of a short cfg5 bench, then the call-I --set full captures
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/m_suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/m_rc.txt
tail -3 gpurun_out/m_suite.log
timeout 1200 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo "bench rc=$?" >> gpurun_out/m_rc.txt
tail -1 gpurun_out/m_bench.json | cut -c1-600
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; echo "ref rc=$?" >> gpurun_out/m_rc.txt
SHORT="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --extra ,"
timeout 600 $SHORT > gpurun_out/m_short_plain.json 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_cfg5.csv $SHORT > gpurun_out/m_ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/m_rc.txt
bash tools/gpu_r02i.sh
cat gpurun_out/m_rc.txt gpurun_out/i_rc.txt
exit 0
