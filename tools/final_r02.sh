#!/bin/bash
# round-2 measurement set at HEAD (under gpurun): GPU tests, smoke, the bench
# line, cfg4 from a thermalized start, cfg5 with its CPU leg and on 1-8
# strips, the reference arm, the bench launch list and full captures of the
# hot kernels (resident CG, cfg2 D^dag D, the decomposed lattice's marching pass).
set -u
O=gpurun_out/final_r02
mkdir -p $O/cfg5_strips
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
tail -3 $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
python bench.py > $O/bench.log 2>&1; grep '^{' $O/bench.log > $O/bench_r02.json
python bench.py --workload cfg4 --therm 20 --steps 5 --warmup 3 > $O/cfg4.log 2>&1; grep '^{' $O/cfg4.log > $O/bench_cfg4_r02.json
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
ncu --set full --clock-control none --import-source on -k regex:k_cg_resblk -c 1 \
  -o $O/ncu_resblk python tools/prof_kernels.py cg > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_resblk.ncu-rep > $O/ncu_full_k_cg_resblk_r02.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_normal_tma -c 1 \
  -o $O/ncu_tma python tools/prof_kernels.py stencil > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_tma.ncu-rep > $O/ncu_full_k_normal_tma_r02.txt 2>&1
SCH_NO_CG_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_dd_march -s 6 -c 1 \
  -o $O/ncu_dd_march_p python tools/prof_dd.py local 1 > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_dd_march_p.ncu-rep > $O/ncu_dd_march_p.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_dd_march -s 2 -c 1 \
  -o $O/ncu_dd_march_plain python tools/prof_dd.py local 1 normal > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_dd_march_plain.ncu-rep > $O/ncu_dd_march_plain.txt 2>&1
python tools/dd_traj_breakdown.py 2048 1 local 2>&1 | grep -v -i warn > $O/dd_traj_breakdown.txt
head -6 $O/ncu_full_k_cg_resblk_r02.txt
for f in bench_r02 bench_cfg4_r02 bench_cfg5_r02 reference_arm_r02; do echo $f; python -c "
import json; d=json.load(open('$O/$f.json')); print({k: d.get(k) for k in ['value','ms_per_step','e2e','cpu_baseline','cg','trajectory']})" 2>&1 | cut -c1-700; done
