#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02b
mkdir -p $O
python -m pytest tests/test_gpu_dd.py -q -m gpu -k "device_heatbath" -p no:cacheprovider > $O/pytest_dd.txt 2>&1
python tools/paper_point_check.py profiles/r02/paper_scale/therm_32x32.cfg \
  nested-fg 0.064 4 5stage-fg 0.064 4 nested-fg 0.064 32 nested-fg 0.04 32 nested-fg 0.064 200 \
  > $O/paper_point.txt 2>&1
SCH_NO_CG_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/dd_launches.csv \
  python tools/prof_dd.py local 1 > /dev/null 2>&1
SCH_NO_CG_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_normal_tile -s 8 -c 1 \
  -o $O/ncu_dd_tile python tools/prof_dd.py local 1 > /dev/null 2>&1
SCH_NO_CG_GRAPH=1 ncu --set full --clock-control none -k regex:k_dd_update -s 4 -c 1 \
  -o $O/ncu_dd_update python tools/prof_dd.py local 1 > /dev/null 2>&1
SCH_RESBLK_XS=6 ncu --set full --clock-control none -k regex:k_cg_resblk -c 1 \
  -o $O/ncu_resblk_xs6 python tools/time_kernels.py cg 16 8192 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:k_cg_cluster_tx -c 1 \
  -o $O/ncu_cluster_tx python tools/time_kernels.py cg 64 1024 > /dev/null 2>&1
ls $O; cat $O/*.txt
