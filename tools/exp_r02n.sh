#!/bin/bash
# Round-2 experiment: deferred solution update in the marching stencil pass (320 B/site/iteration)
set -u
O=gpurun_out/exp_r02n
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5" > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"; }
SCH_DD_DEFER=0 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_nodefer.log 2>&1; show $O/cfg5_nodefer.log nodefer
for v in 32 22 42 23; do
  SCH_DD_MARCH_V=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_v$v.log 2>&1; show $O/cfg5_v$v.log v$v
done
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py launches $O/dd_launches.csv | head -12
