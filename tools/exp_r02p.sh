#!/bin/bash
# Round-2 experiment: per-lane cp.async shared-memory ring for the marching pass (NS slots per warp)
set -u
O=gpurun_out/exp_r02p
mkdir -p $O
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), round(d['roofline']['frac'],3), d['cg']['iterations'], d['cg']['ms_per_iteration'], d['cg']['rel_residual'], round(d['trajectory']['ms']))"; }
SCH_DD_MARCH_V=403 SCH_DD_MARCH_V0=404 timeout 900 python -m pytest tests/test_gpu_dd.py -q -m gpu -x -p no:cacheprovider > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
for v in 402 602 403 304 404; do
  SCH_DD_MARCH_V=$v SCH_DD_MARCH_V0=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_defer_v$v.log 2>&1; show $O/cfg5_defer_v$v.log defer_v$v
done
for v in 403 503 404 602; do
  SCH_DD_DEFER=0 SCH_DD_MARCH_V=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_nodefer_v$v.log 2>&1; show $O/cfg5_nodefer_v$v.log nodefer_v$v
done
