#!/bin/bash
# Round-2 experiment: L2 bulk prefetch (cp.async.bulk.prefetch.L2) ahead of the marching pass's register ring
set -u
O=gpurun_out/exp_r02o
mkdir -p $O
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), round(d['roofline']['frac'],3), d['cg']['ms_per_iteration'], round(d['trajectory']['ms']))"; }
for pd in 4 8 16; do
for v in 22 32 23; do
  SCH_DD_MARCH_PD=$pd SCH_DD_MARCH_V=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_pd${pd}_v$v.log 2>&1; show $O/cfg5_pd${pd}_v$v.log defer_pd${pd}_v$v
done
SCH_DD_DEFER=0 SCH_DD_MARCH_PD=$pd python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_nodefer_pd${pd}.log 2>&1; show $O/cfg5_nodefer_pd${pd}.log nodefer_pd${pd}_v42
SCH_DD_DEFER=0 SCH_DD_MARCH_PD=$pd SCH_DD_MARCH_V=22 SCH_DD_MARCH_V0=22 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_nodefer_pd${pd}_22.log 2>&1; show $O/cfg5_nodefer_pd${pd}_22.log nodefer_pd${pd}_v22
done
