"""Integrator invariants of the reference test-suite, through the GPU path:
inversion counting per macro step and per trajectory
(test_integrators.py:175-191), free-field exactness of every scheme
(:194-201), momentum-flip reversibility of every scheme (:204-213,
test_acceptance.py:178-195) and the HMC exactness identity
<exp(-dH)> = 1 on the thermalized 8x8 configuration (test_acceptance.py)."""

import math

import numpy as np
import pytest
import torch

from conftest import BETA, M0, TOL

pytestmark = pytest.mark.gpu


def _fixtures():
    """q4 / eta4 exactly as the reference conftest draws them."""
    from oracle import schwinger_oracle as O
    rng = O.make_rng(20240401, 0)
    q4 = 0.3 * rng.standard_normal((2, 4, 4))
    rng = O.make_rng(20240401, 0)
    rng.standard_normal((2, 4, 4))
    eta4 = 0.1 * (rng.standard_normal((4, 4, 2)) + 1j * rng.standard_normal((4, 4, 2)))
    return q4, eta4


def _state(sw, q, eta, p=None, beta=BETA, exact=False, tol=TOL):
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.integrators import MdState
    if p is None:
        p = O.sample_momenta(O.make_rng(101, 3), q.shape[-2], q.shape[-1])
    return MdState(q=np.array(q), p=np.array(p), eta=np.array(eta), beta=beta, m0=M0, tol=tol,
                   exact_solves=exact)


def test_inversions_per_macro_step_and_trajectory():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.integrators import (INVERSIONS_PER_STEP, SCHEMES, IntegratorSpec,
                                                   integrate_trajectory)
    q4, eta4 = _fixtures()
    for scheme, expected in INVERSIONS_PER_STEP.items():
        st = _state(sw, q4, eta4, exact=True)
        m = IntegratorSpec(scheme, 0.1).micro_steps()
        SCHEMES[scheme](st, 0.1, m, 1 / 72)
        assert st.counter.count == expected, scheme
    st = _state(sw, q4, eta4, exact=True)
    res = integrate_trajectory(st, IntegratorSpec("leapfrog", 0.05), 2.0)
    assert (res.n_steps, res.inversions) == (40, 160)
    st = _state(sw, q4, eta4, exact=True)
    res = integrate_trajectory(st, IntegratorSpec("5stage", 0.0294), 2.0)
    assert res.n_steps == 68 and res.inversions == 408
    assert math.isclose(res.realized_tau, 68 * 0.0294)


def test_free_field_every_scheme_is_exact():
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.hmc import hamiltonian
    from paper_1512_03812_b200.integrators import SCHEME_IDS, IntegratorSpec, integrate_trajectory
    q = O.hot_start(O.make_rng(31, 0), 4, 4)
    eta = np.zeros((4, 4, 2), complex)
    for scheme in SCHEME_IDS:
        st = _state(sw, q, eta, beta=0.0)
        h0 = float(hamiltonian(st))
        integrate_trajectory(st, IntegratorSpec(scheme, 0.25), 2.0)
        assert abs(float(hamiltonian(st)) - h0) <= 1e-13, scheme


@pytest.mark.parametrize("tau", [0.5, 2.0])
def test_reversibility_every_scheme(tau):
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    from paper_1512_03812_b200.integrators import SCHEME_IDS, IntegratorSpec, integrate_trajectory
    q4, eta4 = _fixtures()
    p0 = O.sample_momenta(O.make_rng(600, 0), 4, 4)
    for scheme in SCHEME_IDS:
        st = _state(sw, q4, eta4, p=p0)
        spec = IntegratorSpec(scheme, 0.05)
        integrate_trajectory(st, spec, tau)
        st.flip_momenta()
        integrate_trajectory(st, spec, tau)
        err = float(np.max(np.abs(O.wrap_angles(st.q.cpu().numpy() - q4))))
        assert err < 1e-10, (scheme, err)


def test_hmc_exactness_identity_on_thermalized_8x8(therm8):
    """E[exp(-dH)] = 1 within three standard errors, the reference's setting
    (leapfrog, h = 0.1, tau = 2, beta = 1, m0 = -0.231367, tol 1e-12) on an
    ensemble: 32 chains started from the thermalized 8x8 configuration, six
    HMC updates each (192 trajectories; the reference runs 200 on one chain)."""
    import paper_1512_03812_b200 as sw
    B = 32
    cfg = sw.HmcConfig(L=8, T=8, beta=BETA, m0=M0, tau=2.0, h=0.1, scheme="leapfrog",
                       cg_tol=1e-12)
    d = sw.NumpyDeviceRng(seed=808, n_chains=B)
    q = torch.as_tensor(np.broadcast_to(therm8, (B,) + therm8.shape).copy(), device="cuda")
    e = []
    for _ in range(6):
        q, st = sw.hmc_update_ensemble(q, cfg, device_rng=d)
        e.append(np.exp(-st.dh))
    e = np.concatenate(e)
    se = e.std(ddof=1) / math.sqrt(e.size)
    assert abs(e.mean() - 1.0) <= 3.0 * se, (e.mean(), se)
