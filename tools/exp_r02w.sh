#!/bin/bash
# Record of a round-2 experiment (the TMA-ring variant it selects was removed afterwards: no gain).
# Round-2: marching pass with a per-warp TMA ring (cp.async.bulk + one mbarrier per slot) vs the register ring
set -u
O=gpurun_out/exp_r02w
mkdir -p $O
SCH_DD_MARCH_V=603 timeout 900 python -m pytest tests/test_gpu_dd.py -q -m gpu -x -p no:cacheprovider > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['cg']['iterations'], d['cg']['ms_per_iteration'], d['cg']['rel_residual'], round(d['trajectory']['ms']))"; }
for v in 0 402 602 802 403 603 404 604; do
  SCH_DD_MARCH_V=$v python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu > $O/cfg5_v$v.log 2>&1; show $O/cfg5_v$v.log v$v
done
