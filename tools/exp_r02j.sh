#!/bin/bash
# Record of a round-2 experiment (profiles/r02/README.md).  Variant switches it sets
# that lost their measurement were removed afterwards (the code is in git history).
set -u
O=gpurun_out/exp_r02j
mkdir -p $O
python tools/variant_dump.py 16 4096 $O/base.npz
SCH_RESBLK_MB=1 python tools/variant_dump.py 16 4096 $O/mb.npz
python tools/variant_dump.py --compare $O/base.npz $O/mb.npz
rm -f $O/*.npz
for v in 0 1 0 1; do SCH_RESBLK_MB=$v python tools/time_kernels.py cg 16 8192; done
SCH_RESBLK_MB=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
SCH_RESBLK_MB=1 python bench.py --steps 5 --warmup 3 --no-cpu --no-stencil --no-compare --no-e2e > $O/bench_mb.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu --no-stencil --no-compare --no-e2e > $O/bench_base.log 2>&1
for f in bench_mb bench_base; do echo $f; grep '^{' $O/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'])"; done
SCH_RESBLK_MB=1 ncu --set full --clock-control none -k regex:k_cg_resblk -c 1 -o $O/ncu_mb python tools/prof_kernels.py cg > /dev/null 2>&1
python tools/ncu_summary.py report $O/ncu_mb.ncu-rep | head -24
