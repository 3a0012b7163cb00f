#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02f
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dd.py -q -m gpu -x -p no:cacheprovider > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
for v in 0 1; do
  SCH_DD_TMA2D=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_t$v.log 2>&1
  echo "tma2d=$v"; grep '^{' $O/cfg5_t$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"
done
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py launches $O/dd_launches.csv | head -10
SCH_NO_CG_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_dd_tma2d -s 4 -c 1 \
  -o $O/ncu_dd_tma2d python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_dd_tma2d.ncu-rep | head -24
bash tools/exp_r02e.sh
