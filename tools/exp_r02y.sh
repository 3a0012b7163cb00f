#!/bin/bash
# Record of a round-2 experiment (the graph cache it measured was reverted: no gain).
# Round-2: instantiated WHILE graphs of the decomposed CG kept per buffer set: DD tests, cfg5 line, trajectory breakdown
set -u
O=gpurun_out/exp_r02y
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py tests/test_gpu_quenched.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5 or strip" > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['cg']['iterations'], d['cg']['ms_per_iteration'], d['cg']['rel_residual'], round(d['trajectory']['ms']), repr(d['trajectory']['dh']))"; }
for i in 1 2; do python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu > $O/cfg5.log 2>&1; show $O/cfg5.log cached; done
python bench.py --workload cfg5 --strips 4 --transport p2p --steps 5 --warmup 3 --no-cpu > $O/cfg5_p2p.log 2>&1; show $O/cfg5_p2p.log cached_p2p4
python tools/dd_traj_breakdown.py 2048 1 local 2>&1 | grep -v -i warn | head -3
