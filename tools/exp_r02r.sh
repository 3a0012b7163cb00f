#!/bin/bash
# Round-2: full ncu captures of the marching pass (CG stencil pass and D^dag D) on cfg5's lattice
set -u
O=gpurun_out/exp_r02r
mkdir -p $O
SCH_NO_CG_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_dd_march -s 6 -c 1 \
  -o $O/ncu_dd_march_p python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_dd_march_p.ncu-rep | head -30
ncu --set full --clock-control none --import-source on -k regex:k_dd_march -s 2 -c 1 \
  -o $O/ncu_dd_march_plain python tools/prof_dd.py local 1 normal > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_dd_march_plain.ncu-rep | head -30
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py launches $O/dd_launches.csv | head -12
