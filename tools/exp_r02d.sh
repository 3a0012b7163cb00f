#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dd.py -q -m gpu -x -p no:cacheprovider > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
for v in "SCH_DD_MARCH=0 SCH_DD_TILE_PF=0" "SCH_DD_MARCH=0 SCH_DD_TILE_PF=1" "SCH_DD_MARCH=5 SCH_DD_TILE_PF=1"; do
  env $v python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5.log 2>&1
  echo "$v"; grep '^{' $O/cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['cg'], d['trajectory']['ms'])"
done
for c in 1024 2048 8192; do
  python bench.py --chains $c --steps 5 --warmup 3 --no-cpu --no-stencil --no-compare --no-e2e > $O/cfg3_$c.log 2>&1
  echo "chains $c"; grep '^{' $O/cfg3_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])"
done
python bench.py --chains 1024 --streams 2 --steps 5 --warmup 3 --no-cpu --no-stencil --no-compare --no-e2e > $O/cfg3_1024s2.log 2>&1
echo "chains 1024 streams 2"; grep '^{' $O/cfg3_1024s2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
