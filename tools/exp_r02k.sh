#!/bin/bash
# Round-2 experiment: the warp-marching stencil pass of the decomposed lattice
# (csrc/march.cuh) against the TMA 2-D tile kernel, variants PF x CTAs/SM.
set -u
O=gpurun_out/exp_r02k
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5" > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"; }
SCH_DD_MARCH=0 python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_tma2d.log 2>&1; show $O/cfg5_tma2d.log tma2d
for v in 23 14 24 22 33 32 42; do
  SCH_DD_MARCH_V=$v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5_v$v.log 2>&1; show $O/cfg5_v$v.log v$v
done
