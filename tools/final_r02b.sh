#!/bin/bash
# round-2 measurement set at HEAD after the marching stencil pass (under
# gpurun): GPU tests, smoke, the bench line, cfg5 with its CPU leg, cfg5 on
# 1-8 strips, the reference arm, the bench launch list.
set -u
O=gpurun_out/final_r02b
mkdir -p $O/cfg5_strips
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.log 2>&1; grep '^{' $O/bench.log > $O/bench_r02.json
python bench.py --workload cfg5 --steps 5 --warmup 3 > $O/cfg5.log 2>&1; grep '^{' $O/cfg5.log > $O/bench_cfg5_r02.json
for s in 1 2 4 8; do for tr in local p2p; do
  python bench.py --workload cfg5 --strips $s --transport $tr --steps 5 --warmup 3 --no-cpu > $O/cfg5_s${s}_$tr.log 2>&1
  grep '^{' $O/cfg5_s${s}_$tr.log > $O/cfg5_strips/cfg5_s${s}_$tr.json
done; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.log 2>&1; grep '^{' $O/ref.log > $O/reference_arm_r02.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-stencil --no-compare > /dev/null 2>&1
python tools/ncu_summary.py launches $O/bench_launches.csv > $O/bench_launches_summary.txt 2>&1
head -8 $O/bench_launches_summary.txt
for f in bench_r02 bench_cfg5_r02 reference_arm_r02; do echo $f; python -c "
import json; d=json.load(open('$O/$f.json')); print({k: d.get(k) for k in ['value','ms_per_step','e2e','cg','roofline']})" 2>&1 | cut -c1-900; done
for f in $O/cfg5_strips/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f'.split('/')[-1], round(d['value']), d['cg']['ms_per_iteration'], round(d['trajectory']['ms']), repr(d['trajectory']['dh']))"; done
