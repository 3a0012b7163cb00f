#!/bin/bash
# Round-2 experiment: launch list of the decomposed CG with the marching stencil pass
set -u
O=gpurun_out/exp_r02l
mkdir -p $O
for v in 42 22 23; do
SCH_DD_MARCH_V=$v SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches_v$v.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
echo "== v$v"; python tools/ncu_summary.py launches $O/dd_launches_v$v.csv | head -12
done
