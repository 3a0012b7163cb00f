#!/bin/bash
# Paper-scale reproduction on the GPU (Table 1
# and Figs. 1-2): the reference's benchmark point (HmcConfig defaults:
# 32x32, beta 1, m0 -0.231367, tau 2, 200 samples), a thermalized start from
# the harness, acceptance tuning to 90 % per scheme (inversions per
# trajectory = Table 1), the |dH| step-size sweep, and the reference suite's
# paper-scale qualitative criteria.
#
# Two passes: the paper's CG tolerance 1e-12, and 1e-10.  At 1e-12 the
# batched (batch-global) solves of the force-gradient schemes' Z pair sit on
# the float64 attainable-accuracy floor (best relative residual 1.0-3e-12
# after 10000 iterations) — the reference itself raises SolverError there on
# the same inputs (profiles/r02/paper_scale/README.md) — so Table 1 is
# completed at 1e-10.
#   bash tools/paper_scale.sh [outdir]        (run under gpurun)
set -euo pipefail
OUT=${1:-gpurun_out/paper_scale}
mkdir -p "$OUT"
H="python -m paper_1512_03812_b200.harness"
step() {   # name, log, command...
  local name=$1 log=$2; shift 2
  local t0=$SECONDS
  "$@" 2>&1 | tee "$log"
  echo "$name $((SECONDS - t0)) s" | tee -a "$log"
}
for tol in 1e-12 1e-10; do
  cat > "$OUT/exp_$tol.cfg" <<CFG
# the paper's benchmark point: HmcConfig defaults (32x32, beta 1, m0 -0.231367, tau 2)
n_samples = 200
cg_tol = $tol
gauge_config = $OUT/therm_32x32.cfg
schemes = leapfrog,5stage,nested-5stage,5stage-fg,fg-approx,nested-fg,adapted-nested-fg,11stage
h_min = 0.005
h_max = 0.15
target = 0.9
h_grid = 0.02,0.03,0.04,0.05,0.064
CFG
done
# the committed thermalized configuration of the first run, when present
if [ ! -f "$OUT/therm_32x32.cfg" ] && [ -f profiles/r02/paper_scale/therm_32x32.cfg ]; then
  cp profiles/r02/paper_scale/therm_32x32.cfg* "$OUT/"
fi
if [ ! -f "$OUT/therm_32x32.cfg" ]; then
  step thermalize "$OUT/thermalize.log" $H thermalize --config "$OUT/exp_1e-12.cfg" --out "$OUT/therm_32x32.cfg"
fi
for tol in 1e-12 1e-10; do
  step "tune-acceptance tol $tol" "$OUT/tune_$tol.log" $H tune-acceptance --config "$OUT/exp_$tol.cfg" --out "$OUT/table1_tuned_$tol.csv"
  step "sweep-dh tol $tol" "$OUT/sweep_$tol.log" $H sweep-dh --config "$OUT/exp_$tol.cfg" --out "$OUT/fig1_sweep_$tol.csv"
done
SCHWINGER_PAPER_SCALE=1 SCHWINGER_PAPER_TOL=1e-10 python -m pytest tests/test_gpu_paper_claims.py -m gpu -q -s \
  -k paper_scale -p no:cacheprovider 2>&1 | tee "$OUT/qualitative_1e-10.txt" | tail -30
