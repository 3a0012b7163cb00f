#!/bin/bash
# Round-2: shuffle t-faces in the 64^2 cluster CG: parity tests, timing, cfg4 line
set -u
O=gpurun_out/exp_r02x
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
python tools/time_kernels.py cg 64 1024
python tools/time_kernels.py cg 64 148
python bench.py --workload cfg4 --therm 20 --steps 5 --warmup 3 --no-cpu > $O/cfg4.log 2>&1
grep '^{' $O/cfg4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['config'].get('cg_iterations_per_solve'))"
