#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
# latency vs throughput of the resident / cluster CG: ns per chain-iteration
# at B = one chain, one wave, many waves
set -u
O=gpurun_out/exp_r02e
mkdir -p $O
for b in 1 37 74 148 1024; do python tools/time_kernels.py cg 64 $b; done > $O/lat64.txt 2>&1
for b in 1 148 592 1184 8192; do python tools/time_kernels.py cg 16 $b; done > $O/lat16.txt 2>&1
cat $O/*.txt
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches_head.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py launches $O/dd_launches_head.csv | head -12
python bench.py --workload cfg5 --steps 5 --warmup 2 > $O/cfg5_head.log 2>&1
grep '^{' $O/cfg5_head.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['cg'], d['trajectory'], d['cpu_baseline'])"
