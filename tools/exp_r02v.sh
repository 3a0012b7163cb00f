#!/bin/bash
# Round-2: programmatic dependent launches between the decomposed CG's kernels: DD tests, cfg5 A/B
set -u
O=gpurun_out/exp_r02v
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dd.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "dd or cfg5" > $O/pytest_dd.txt 2>&1
tail -3 $O/pytest_dd.txt
show() { grep '^{' $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$2', round(d['value']), d['cg']['iterations'], d['cg']['ms_per_iteration'], d['cg']['rel_residual'], round(d['trajectory']['ms']), repr(d['trajectory']['dh']))"; }
for i in 1 2; do
python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu > $O/cfg5_pdl.log 2>&1; show $O/cfg5_pdl.log pdl
SCH_NO_PDL=1 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu > $O/cfg5_nopdl.log 2>&1; show $O/cfg5_nopdl.log nopdl
done
python bench.py --workload cfg5 --strips 4 --transport p2p --steps 5 --warmup 3 --no-cpu > $O/cfg5_pdl_p2p.log 2>&1; show $O/cfg5_pdl_p2p.log pdl_p2p4
