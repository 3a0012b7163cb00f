#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02i
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5" > $O/pytest_dd.txt 2>&1
tail -2 $O/pytest_dd.txt
python bench.py --workload cfg5 --steps 5 --warmup 2 > $O/cfg5.log 2>&1
grep '^{' $O/cfg5.log > $O/bench_cfg5_r02.json
grep '^{' $O/cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py launches $O/dd_launches.csv 2>/dev/null | head -10
