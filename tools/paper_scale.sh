#!/bin/bash
# Paper-scale reproduction on the GPU (Table 1
# and Figs. 1-2): the reference's benchmark point (HmcConfig defaults:
# 32x32, beta 1, m0 -0.231367, tau 2, CG tol 1e-12, 200 samples), a
# thermalized start from the harness, acceptance tuning to 90 % per scheme
# (inversions per trajectory = Table 1), the |dH| step-size sweep, and the
# reference suite's paper-scale qualitative criteria.
#   bash tools/paper_scale.sh [outdir]        (run under gpurun)
set -euo pipefail
OUT=${1:-gpurun_out/paper_scale}
mkdir -p "$OUT"
cat > "$OUT/exp.cfg" <<CFG
# the paper's benchmark point: HmcConfig defaults (32x32, beta 1, m0 -0.231367, tau 2)
n_samples = 200
gauge_config = $OUT/therm_32x32.cfg
schemes = leapfrog,5stage,nested-5stage,5stage-fg,fg-approx,nested-fg,adapted-nested-fg,11stage
h_min = 0.005
h_max = 0.15
target = 0.9
h_grid = 0.02,0.03,0.04,0.05,0.064
CFG
H="python -m paper_1512_03812_b200.harness"
step() {   # name, log, command...
  local name=$1 log=$2; shift 2
  local t0=$SECONDS
  "$@" 2>&1 | tee "$log"
  echo "$name $((SECONDS - t0)) s" | tee -a "$log"
}
step thermalize "$OUT/thermalize.log" $H thermalize --config "$OUT/exp.cfg" --out "$OUT/therm_32x32.cfg"
step tune-acceptance "$OUT/tune.log" $H tune-acceptance --config "$OUT/exp.cfg" --out "$OUT/table1_tuned.csv"
step sweep-dh "$OUT/sweep.log" $H sweep-dh --config "$OUT/exp.cfg" --out "$OUT/fig1_sweep.csv"
SCHWINGER_PAPER_SCALE=1 python -m pytest tests/test_gpu_paper_claims.py -m gpu -q -s -k paper_scale \
  2>&1 | tee "$OUT/qualitative.txt" | tail -20
