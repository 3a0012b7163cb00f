#!/bin/bash
# Round-2: the parallel walk of one long NumPy stream (cfg5's heatbath) and the libm-exact tail:
# all GPU tests, trajectory breakdown, cfg5 line
set -u
O=gpurun_out/exp_r02u
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/pytest.txt 2>&1
tail -4 $O/pytest.txt
python tools/dd_traj_breakdown.py 2048 1 local 2>&1 | grep -v -i warn | head -12 | tee $O/dd_traj_breakdown.txt
python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu > $O/cfg5.log 2>&1
grep '^{' $O/cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['cg']['ms_per_iteration'], d['trajectory']['ms'], d['trajectory']['dh'])"
