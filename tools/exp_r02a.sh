#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
# round-2 kernel-variant experiment (run under gpurun): resident CG with x in
# shared memory (SCH_RESBLK_XS), cluster CG shapes (SCH_CLUSTER), cluster
# placement probe, parity of every variant against the default.
set -u
O=gpurun_out/exp_r02a
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/micro/cluster_place tools/micro/cluster_place.cu
for a in "8 2" "8 3" "4 1" "2 2"; do tools/micro/cluster_place $a; done > $O/cluster_place.txt 2>&1
python tools/variant_dump.py 16 2048 $O/r16_base.npz
for v in 4 6; do
  SCH_RESBLK_XS=$v python tools/variant_dump.py 16 2048 $O/r16_xs$v.npz
  python tools/variant_dump.py --compare $O/r16_base.npz $O/r16_xs$v.npz >> $O/parity.txt
done
python tools/variant_dump.py 64 64 $O/r64_base.npz
for v in 8 83; do
  SCH_CLUSTER=$v python tools/variant_dump.py 64 64 $O/r64_c$v.npz
  python tools/variant_dump.py --compare $O/r64_base.npz $O/r64_c$v.npz >> $O/parity.txt
done
for v in 0 4 6; do
  SCH_RESBLK_XS=$v python tools/time_kernels.py cg 16 8192
done > $O/time16.txt 2>&1
for v in 4 8 83; do
  SCH_CLUSTER=$v python tools/time_kernels.py cg 64 1024
done > $O/time64.txt 2>&1
rm -f $O/*.npz
python bench.py --workload cfg5 --steps 5 --warmup 2 --no-cpu > $O/cfg5.log 2>&1
python bench.py --workload cfg4 --steps 3 --warmup 3 --no-cpu --no-e2e --no-stencil > $O/cfg4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_normal_tile -s 8 -c 2 \
  -o $O/ncu_dd_tile python tools/prof_dd.py local 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_dd_update -s 4 -c 1 \
  -o $O/ncu_dd_update python tools/prof_dd.py local 1 > /dev/null 2>&1
cat $O/*.txt; tail -c 1500 $O/cfg5.log; tail -c 1500 $O/cfg4.log
