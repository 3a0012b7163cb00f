#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dd.py -q -m gpu -x -p no:cacheprovider > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
for v in 0 1 5 6 7; do
  SCH_DD_MARCH=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_v$v.log 2>&1
done
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
for f in $O/cfg5_v*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"; done
