"""Forces against finite differences of the actions, on the GPU path — the
reference's own checks (test_fermion.py:225-236, test_gauge.py:52-69) — with
all 2 x 32 perturbed configurations of a 4x4 lattice evaluated as one batch."""

import numpy as np
import pytest
import torch

from conftest import BETA, M0, TOL

pytestmark = pytest.mark.gpu


def _q4_eta4():
    from oracle import schwinger_oracle as O
    rng = O.make_rng(20240401, 0)
    q4 = 0.3 * rng.standard_normal((2, 4, 4))
    eta4 = 0.1 * (rng.standard_normal((4, 4, 2)) + 1j * rng.standard_normal((4, 4, 2)))
    return q4, eta4


def fd_gradient_batched(action, q, eps):
    """Central differences of action(batch of configurations) -> (B,)."""
    plus, minus = [], []
    for idx in np.ndindex(q.shape):
        qp, qm = q.copy(), q.copy()
        qp[idx] += eps
        qm[idx] -= eps
        plus.append(qp)
        minus.append(qm)
    v = action(np.stack(plus + minus))
    n = len(plus)
    return ((v[:n] - v[n:]) / (2 * eps)).reshape(q.shape)


def test_fermion_force_matches_fd():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import fermion as F
    q4, eta4 = _q4_eta4()
    op = sw.WilsonDirac(q4, M0)
    chi, xi, _ = F.chi_xi(op, eta4, TOL)
    force = F.fermion_force(op, chi, xi).cpu().numpy()

    def action(qs):
        opb = sw.WilsonDirac(qs, M0)
        eta = np.broadcast_to(eta4, (qs.shape[0],) + eta4.shape).copy()
        return F.fermion_action(opb, eta, TOL, stop="per_chain").cpu().numpy()

    ref = fd_gradient_batched(action, q4, 1e-5)
    assert np.max(np.abs(force - ref)) < 1e-6


def test_fermion_force_zero_without_pseudofermion():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import fermion as F
    q4, _ = _q4_eta4()
    op = sw.WilsonDirac(q4, M0)
    zero = np.zeros((4, 4, 2), complex)
    assert bool((F.fermion_force(op, zero, zero) == 0.0).all())


def test_gauge_force_matches_fd_and_closed_forms():
    import paper_1512_03812_b200 as sw
    q4, _ = _q4_eta4()
    f = sw.gauge_force(q4, BETA).cpu().numpy()
    ref = fd_gradient_batched(lambda qs: sw.gauge_action(qs, BETA).cpu().numpy(), q4, 1e-5)
    assert np.max(np.abs(f - ref)) < 1e-8
    # beta factorisation (test_gauge.py:68-69)
    assert np.allclose(sw.gauge_force(q4, 1.7).cpu().numpy(),
                       1.7 * sw.gauge.gauge_force_raw(q4).cpu().numpy())
    # a single excited link (test_gauge.py:52-59)
    q = np.zeros((2, 4, 4))
    q[0, 1, 1] = 0.5
    g = sw.gauge_force(q, BETA).cpu().numpy()
    assert np.isclose(g[0, 1, 1], 2 * BETA * np.sin(0.5))
    assert abs(g[0, 3, 3]) < 1e-15
