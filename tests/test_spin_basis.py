"""The sigma1-diagonal spin basis of the resident CG engines (block_stencil.cuh
SiteBlockRot, resident_col.cuh ROT), checked on CPU against the oracle.

The kernels solve D'^dag D' x' = T b with D' = H D H, T = [[1,1],[1,-1]],
H = T/sqrt2, and return x = T x' / 2.  This restates their per-site hop
formulas in NumPy (x hops read and write one spin component; t hops are the
reference D^dag's for D and vice versa) and checks them against the oracle's
D / D^dag / D^dag D (fermion.py:101-131), so the basis algebra is pinned
independently of the GPU parity tests, which exercise the same path through
the C ABI.
"""

import numpy as np
import pytest

from oracle import schwinger_oracle as O


def _spin_rot(v):          # v' = T v
    return np.stack([v[..., 0] + v[..., 1], v[..., 0] - v[..., 1]], axis=-1)


def _spin_unrot(v):        # x = T x' / 2
    return 0.5 * _spin_rot(v)


def _fwd(a, mu):           # a(n + mu)
    return np.roll(a, -1, axis=-2 + mu)


def _bwd(a, mu):           # a(n - mu)
    return np.roll(a, 1, axis=-2 + mu)


def rotated_dirac(U, v, m0, dagger=False):
    """D' v' (or D'^dag v') with the kernel's formulas.  U: (..., 2, L, T)
    complex links, v: (..., L, T, 2) in the rotated basis.  Links prescaled as
    in the kernels: u0 by -1, u1 by -1/2."""
    u0, u1 = -U[..., 0, :, :], -0.5 * U[..., 1, :, :]
    v0, v1 = v[..., 0], v[..., 1]
    diag = 2.0 + m0
    o0, o1 = diag * v0, diag * v1
    # x: forward hop lands in component 1 (D) / 0 (D^dag); backward in the other
    if not dagger:
        o1 = o1 + u0 * _fwd(v1, 0)
        o0 = o0 + _bwd(np.conj(u0) * v0, 0)
    else:
        o0 = o0 + u0 * _fwd(v0, 0)
        o1 = o1 + _bwd(np.conj(u0) * v1, 0)
    # t: D' uses the reference D^dag's projectors and coefficients
    #   D:     f = v0 - i v1 -> (h, +i h);  b = conj(u1) (v0 + i v1) -> (h, -i h)
    #   D^dag: f = v0 + i v1 -> (h, -i h);  b = conj(u1) (v0 - i v1) -> (h, +i h)
    s = 1.0 if not dagger else -1.0
    hf = u1 * _fwd(v0 - s * 1j * v1, 1)
    hb = _bwd(np.conj(u1) * (v0 + s * 1j * v1), 1)
    o0 = o0 + hf + hb
    o1 = o1 + s * 1j * hf - s * 1j * hb
    return np.stack([o0, o1], axis=-1)


@pytest.fixture(scope="module")
def field():
    rng = np.random.default_rng(7)
    B, L, T = 3, 8, 6
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, T))
    psi = rng.standard_normal((B, L, T, 2)) + 1j * rng.standard_normal((B, L, T, 2))
    return q, psi


@pytest.mark.parametrize("bc", ["periodic", "antiperiodic"])
@pytest.mark.parametrize("dagger", [False, True])
def test_rotated_dirac_is_h_d_h(field, bc, dagger):
    q, psi = field
    U = O.fermion_links(q, bc)
    ref = O.dirac(U, psi, 0.1, dagger=dagger)
    # D' (T psi) = T (D psi)  <=>  H D H = D' with H = T / sqrt2
    got = rotated_dirac(U, _spin_rot(psi), 0.1, dagger=dagger)
    np.testing.assert_allclose(got, _spin_rot(ref), rtol=0, atol=1e-13 * np.abs(ref).max())


def test_rotated_normal_and_round_trip(field):
    q, psi = field
    U = O.fermion_links(q)
    ref = O.normal_op(U, psi, 0.1)
    vp = _spin_rot(psi)
    got = _spin_unrot(rotated_dirac(U, rotated_dirac(U, vp, 0.1), 0.1, dagger=True))
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    # norms scale by exactly 2 (T^dag T = 2): relative residuals are basis-independent
    assert np.isclose(np.vdot(vp, vp).real, 2 * np.vdot(psi, psi).real, rtol=1e-14)
    np.testing.assert_array_equal(_spin_unrot(_spin_rot(np.array([[1.0 + 2j, 3.0 - 1j]]))),
                                  np.array([[1.0 + 2j, 3.0 - 1j]]))


def test_x_hops_touch_one_component(field):
    """The property the kernels exploit: with the t links zeroed, a unit
    source in one rotated component spreads in x into exactly one component."""
    q, _ = field
    U = O.fermion_links(q)
    U[..., 1, :, :] = 0.0
    src = np.zeros((3, 8, 6, 2), complex)
    src[:, 4, 2, 1] = 1.0
    out = rotated_dirac(U, src, 0.0)   # m0 = -2 would kill the diagonal; use m0 = 0
    out[:, 4, 2, :] -= 2.0 * src[:, 4, 2, :]
    # D: component 1 of n+x feeds component 1 at n (the forward hop), nothing else
    nz = np.argwhere(np.abs(out) > 0)
    assert set(map(tuple, nz[:, 1:])) == {(3, 2, 1)}
