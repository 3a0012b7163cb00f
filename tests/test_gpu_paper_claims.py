"""The paper's integrator claims, checked on the GPU path with the reference
suite's own criteria:

* order of convergence: log-log slope of mean |dH| over 50 samples and four
  step sizes on the thermalized 8x8 configuration (pkg/tests/
  test_acceptance.py:130-156): every cell equal to the reference's own run,
  and at least the published order for each scheme (see the test);
* volume preservation: every scheme's one-step map has a finite-difference
  Jacobian determinant of 1 within 1e-8 (test_integrators.py:216-241);
* the Taylor-approximated force-gradient kick tracks the exact one, gap
  shrinking faster than h^4.7 (test_integrators.py:244-260);
* the inner (gauge-only) flows: leapfrog Richardson ratio ~4 per doubling,
  force-gradient micro flow 4th order in dH, the two flows converge to each
  other (test_integrators.py:135-168).

The reference's hours-scale 32x32 qualitative reproduction (nested below
plain, tuned step-size bands, nested force-gradient cheapest at 90 %
acceptance; test_acceptance.py:219-268) runs with SCHWINGER_PAPER_SCALE=1,
as in the reference (tools/paper_scale.sh records it under profiles/).
"""

import math
import os
from dataclasses import replace

import numpy as np
import pytest

from conftest import BETA, M0, TOL

pytestmark = pytest.mark.gpu

SECOND_ORDER = ("leapfrog", "5stage", "nested-leapfrog", "nested-5stage")
FOURTH_ORDER = ("5stage-fg", "fg-approx", "11stage", "nested-fg", "adapted-nested-fg")


def npy(t):
    return t.detach().cpu().numpy()


def _q4_eta4():
    from oracle import schwinger_oracle as O
    rng = O.make_rng(20240401, 0)
    q4 = 0.3 * rng.standard_normal((2, 4, 4))
    rng = O.make_rng(20240401, 0)
    rng.standard_normal((2, 4, 4))
    eta4 = 0.1 * (rng.standard_normal((4, 4, 2)) + 1j * rng.standard_normal((4, 4, 2)))
    return q4, eta4


def _state(q, eta, p=None, beta=BETA, exact=False):
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.integrators import MdState
    if p is None:
        p = O.sample_momenta(O.make_rng(101, 3), q.shape[-2], q.shape[-1])
    return MdState(q=np.array(q), p=np.array(p), eta=np.array(eta), beta=beta, m0=M0, tol=TOL,
                   exact_solves=exact)


def _wrapped(d):
    return np.mod(d + np.pi, 2 * np.pi) - np.pi


def test_order_of_convergence(therm8, golden):
    """Every (scheme, h) cell of the reference's order test on the GPU path:
    mean |dH| equal to the reference's own run on the same fixture
    (tests/golden/order.npz, tests/golden/make_order_golden.py), the same
    log-log slopes, and each scheme converging at least at its published
    order (2 - 0.2 / 4 - 0.3).  The reference's two-sided bands do not hold
    on this regenerated fixture for the reference itself either (its
    therm_8x8.cfg is missing; on the one regenerated with its thermalize the
    reference measures leapfrog 2.61, 5stage 3.77, force-gradient family
    7.4-8.3: the grid is not in the asymptotic regime), so the test pins
    the GPU to the reference's measured convergence and checks the order
    claim as a lower bound."""
    import paper_1512_03812_b200 as sw
    g = golden("order")
    base = sw.HmcConfig(L=8, T=8, beta=BETA, m0=M0, tau=2.0, n_samples=50)
    slopes, worst = {}, 0.0
    for scheme in SECOND_ORDER + FOURTH_ORDER:
        grid = g[f"{scheme}_h"]
        means = []
        for k, h in enumerate(grid):
            micro = math.ceil(1.0 / h) if scheme in ("nested-fg", "adapted-nested-fg") else None
            cfg = replace(base, scheme=scheme, h=float(h), micro_per_call=micro)
            m = sw.measure_dh(therm8, cfg, sw.make_rng(400, 7), n_samples=50)
            assert m.inversions_per_traj == int(g[f"{scheme}_inv"][k]), (scheme, h)
            # the north_star dH bar (1e-8 absolute) on the mean of 50 |dH|
            assert abs(m.mean_abs - g[f"{scheme}_mean"][k]) <= 1e-8, \
                (scheme, h, m.mean_abs, g[f"{scheme}_mean"][k])
            worst = max(worst, abs(m.mean_abs / g[f"{scheme}_mean"][k] - 1.0))
            means.append(m.mean_abs)
        slopes[scheme] = float(np.polyfit(np.log(grid), np.log(means), 1)[0])
        ref = float(np.polyfit(np.log(grid), np.log(g[f"{scheme}_mean"]), 1)[0])
        assert abs(slopes[scheme] - ref) < 1e-3, (scheme, slopes[scheme], ref)
    print("order-of-convergence slopes:", {k: round(v, 3) for k, v in slopes.items()},
          f"worst relative difference of a mean |dH| cell from the reference: {worst:.1e}")
    for scheme in SECOND_ORDER:
        assert slopes[scheme] >= 2.0 - 0.2, (scheme, slopes[scheme])
    for scheme in FOURTH_ORDER:
        assert slopes[scheme] >= 4.0 - 0.3, (scheme, slopes[scheme])
    assert min(slopes[s] for s in FOURTH_ORDER) > max(slopes["leapfrog"], slopes["nested-leapfrog"])


def test_volume_preservation_jacobian():
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.integrators import SCHEME_IDS, SCHEMES, MdState
    rng = O.make_rng(3, 0)
    q0 = 0.3 * rng.standard_normal((2, 2, 2))
    p0 = O.sample_momenta(rng, 2, 2)
    eta = 0.1 * (rng.standard_normal((2, 2, 2)) + 1j * rng.standard_normal((2, 2, 2)))
    nl = q0.size

    def one_step(z, scheme):
        st = MdState(q=z[:nl].reshape(q0.shape).copy(), p=z[nl:].reshape(q0.shape).copy(),
                     eta=eta, beta=BETA, m0=M0, tol=TOL, exact_solves=True)
        SCHEMES[scheme](st, 0.08, 4, 1 / 72)
        return np.concatenate([npy(st.q).ravel(), npy(st.p).ravel()])

    z0 = np.concatenate([q0.ravel(), p0.ravel()])
    eps = 1e-6
    dets = {}
    for scheme in SCHEME_IDS:
        jac = np.empty((2 * nl, 2 * nl))
        for k in range(2 * nl):
            zp, zm = z0.copy(), z0.copy()
            zp[k] += eps
            zm[k] -= eps
            jac[:, k] = (one_step(zp, scheme) - one_step(zm, scheme)) / (2 * eps)
        dets[scheme] = float(np.linalg.det(jac))
        assert abs(dets[scheme] - 1.0) < 1e-8, (scheme, dets[scheme])
    print("Jacobian determinants - 1:", {k: f"{v - 1:.1e}" for k, v in dets.items()})


def test_fg_approx_tracks_exact_fg(therm8):
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.integrators import SCHEMES
    rng = O.make_rng(77, 0)
    eta = 0.3 * (rng.standard_normal((8, 8, 2)) + 1j * rng.standard_normal((8, 8, 2)))
    p = O.sample_momenta(rng, 8, 8)
    hs = np.array([0.1, 0.05, 0.025])
    gaps = []
    for h in hs:
        a = _state(therm8, eta, p=p)
        SCHEMES["5stage-fg"](a, h, 1, 1 / 72)
        b = _state(therm8, eta, p=p)
        SCHEMES["fg-approx"](b, h, 1, 1 / 72)
        gaps.append(np.max(np.abs(np.concatenate(
            [_wrapped(npy(a.q) - npy(b.q)).ravel(), (npy(a.p) - npy(b.p)).ravel()]))))
    slope = np.polyfit(np.log(hs), np.log(gaps), 1)[0]
    print("fg-approx vs exact FG gap slope:", round(float(slope), 3), gaps)
    assert slope > 4.7, (gaps, slope)


def test_inner_flows_reverse_richardson_and_order():
    from paper_1512_03812_b200.hmc import hamiltonian
    from paper_1512_03812_b200.integrators import inner_fg, inner_leapfrog
    q4, eta4 = _q4_eta4()
    # reversibility of both micro flows
    for flow in (inner_leapfrog, lambda s, h, m: inner_fg(s, h, m, 1 / 72)):
        st = _state(q4, eta4)
        flow(st, 0.4, 5)
        st.flip_momenta()
        flow(st, 0.4, 5)
        assert np.max(np.abs(_wrapped(npy(st.q) - q4))) < 1e-11
    # leapfrog: doubling M shrinks the flow error like M^-2
    diffs = []
    for m in (4, 8, 16):
        a = _state(q4, eta4)
        inner_leapfrog(a, 0.8, m)
        b = _state(q4, eta4)
        inner_leapfrog(b, 0.8, 2 * m)
        diffs.append(np.max(np.abs(_wrapped(npy(a.q) - npy(b.q)))))
    rates = [diffs[i] / diffs[i + 1] for i in range(2)]
    assert all(2.5 < r < 6.0 for r in rates), (diffs, rates)
    # gauge-only force-gradient micro flow: dH converges like delta^4
    errs = []
    for m in (2, 4, 8):
        st = _state(q4, np.zeros((4, 4, 2), complex))
        h0 = float(hamiltonian(st))
        inner_fg(st, 0.8, m, 1 / 72)
        errs.append(abs(float(hamiltonian(st)) - h0))
    slopes = [np.log(errs[i] / errs[i + 1]) / np.log(2) for i in range(2)]
    assert all(3.5 < s < 4.6 for s in slopes), (errs, slopes)
    # the two micro flows agree as M grows
    gaps = []
    for m in (4, 16):
        a = _state(q4, eta4)
        inner_leapfrog(a, 0.5, m)
        b = _state(q4, eta4)
        inner_fg(b, 0.5, m, 1 / 72)
        gaps.append(np.max(np.abs(_wrapped(npy(a.q) - npy(b.q)))))
    assert gaps[1] < gaps[0] / 4


@pytest.mark.skipif(os.environ.get("SCHWINGER_PAPER_SCALE") != "1",
                    reason="32x32, 200-sample tuning of eight schemes; set SCHWINGER_PAPER_SCALE=1")
def test_paper_scale_qualitative():
    """The reference's paper-scale criteria (test_acceptance.py:219-268) on
    the GPU: nested curves below their plain twins at equal h, tuned step
    sizes inside the published bands, and the nested force-gradient pair the
    cheapest in inversions per trajectory at 90 % acceptance."""
    import paper_1512_03812_b200 as sw
    # SCHWINGER_PAPER_TOL: the CG tolerance (the paper's 1e-12 by default).
    # At 1e-12 the batched solves of the force-gradient schemes' Z pair hit
    # the float64 floor on 32x32 at this mass — the reference raises
    # SolverError there too (profiles/r02/paper_scale/README.md) — so the
    # recorded run uses 1e-10.
    tol = float(os.environ.get("SCHWINGER_PAPER_TOL", "1e-12"))
    cfg = sw.HmcConfig(n_thermalize=500, h=0.05, cg_tol=tol)
    q0, _ = sw.thermalize(cfg, sw.make_rng(cfg.seed, 0), on_solver_error="reject")
    pairs = [("leapfrog", "nested-leapfrog"), ("5stage", "nested-5stage"),
             ("5stage-fg", "nested-fg")]
    for h in (0.04, 0.064):
        for plain, nested in pairs:
            mp = sw.measure_dh(q0, replace(cfg, scheme=plain, h=h), sw.make_rng(2000, 1),
                               n_samples=200)
            mn = sw.measure_dh(q0, replace(cfg, scheme=nested, h=h), sw.make_rng(2000, 1),
                               n_samples=200)
            print(f"h={h} {plain} {mp.mean_abs:.4g} {nested} {mn.mean_abs:.4g}")
            assert mn.mean_abs < mp.mean_abs + 2 * (mn.stderr + mp.stderr), (plain, nested, h)

    def tune(scheme, lo, hi):
        for _ in range(24):
            mid = 0.5 * (lo + hi)
            try:
                m = sw.measure_dh(q0, replace(cfg, scheme=scheme, h=mid), sw.make_rng(3000, 5),
                                  n_samples=200)
            except sw.SolverError:   # CG cap on a wild trajectory: h too large
                hi = mid
                continue
            if abs(m.acceptance - 0.9) <= 0.02:
                return mid, m
            if m.acceptance > 0.9:
                lo = mid
            else:
                hi = mid
        return mid, m

    tuned = {}
    for scheme in ("leapfrog", "5stage", "nested-5stage", "5stage-fg", "fg-approx", "nested-fg",
                   "adapted-nested-fg", "11stage"):
        h_star, m = tune(scheme, 0.005, 0.15)
        tuned[scheme] = (h_star, m.inversions_per_traj)
        print(f"tuned {scheme}: h={h_star:.5f} acceptance={m.acceptance:.3f} "
              f"inversions/traj={m.inversions_per_traj}")
    for scheme in ("leapfrog", "5stage", "nested-5stage"):
        assert 0.02 <= tuned[scheme][0] <= 0.04, (scheme, tuned[scheme])
    for scheme in ("5stage-fg", "fg-approx", "nested-fg", "adapted-nested-fg"):
        assert 0.04 <= tuned[scheme][0] <= 0.08, (scheme, tuned[scheme])
    costs = {s: c for s, (_, c) in tuned.items()}
    assert min(costs["nested-fg"], costs["adapted-nested-fg"]) == min(costs.values())
