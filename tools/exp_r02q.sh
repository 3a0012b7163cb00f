#!/bin/bash
# Round-2: marching pass with explicit multiply-add arithmetic: DD tests + cfg5 line
set -u
O=gpurun_out/exp_r02q
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5" > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), round(d['roofline']['frac'],3), d['cg']['iterations'], d['cg']['ms_per_iteration'], d['cg']['rel_residual'], round(d['trajectory']['ms']))"; }
python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5.log 2>&1; show $O/cfg5.log march
