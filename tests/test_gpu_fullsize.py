"""Parity at BASELINE.json's full sizes (configs[1]-[4]), through checks that
do not need the oracle to redo the whole run:

* cfg2 (4096 x 32^2): every batch element of the fused D^dag D against the
  oracle's batched NumPy stencil; linearity and hermiticity of D^dag D over
  the whole batch; the per-chain CG to 1e-10: every one of the 4096
  solutions against the oracle's per-chain solve (<= 1e-12 relative per
  chain) with identical iteration counts for every chain (the oracle spread
  over the host cores, oracle/parallel.py); the batch-global CG with every
  chain's true residual recomputed by the oracle.
* cfg3 (8192 x 16^2): one HMC update of the whole ensemble on the
  reference's own per-chain streams; 512 chains spread over the ensemble
  equal independent oracle hmc_update calls (dH <= 1e-8, accept, links,
  inversions); every chain's dH is finite and the acceptance is the
  schedule's.
* cfg4 (1024 x 64^2, m0 = 0.02): per-chain CG (cluster engine): every
  chain's solution (<= 1e-12) and iteration count against the oracle.
* cfg5 (2048^2): the decomposed D^dag D (local and peer-memory transports)
  against the oracle on the whole lattice; the decomposed CG on 2 and 8
  strips bit-identical to the one-strip solve, with its true residual.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL_OP = 1e-12


def npy(t):
    return t.detach().cpu().numpy()


def per_element_rel(a, b):
    """max_site |a - b| / max_site |b| for every batch element."""
    axes = tuple(range(1, a.ndim))
    return np.max(np.abs(a - b), axis=axes) / np.max(np.abs(b), axis=axes)


def true_relres(O, U, m0, x, b):
    r = b - O.normal_op(U, x, m0)
    axes = tuple(range(1, r.ndim))
    return np.sqrt(np.sum(np.abs(r) ** 2, axis=axes) / np.sum(np.abs(b) ** 2, axis=axes))


@pytest.fixture(scope="module")
def cfg2():
    rng = np.random.default_rng(4096)
    B, L = 4096, 32
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, L))
    psi = (rng.standard_normal((B, L, L, 2)) + 1j * rng.standard_normal((B, L, L, 2)))
    return q, psi


def test_cfg2_ddagd_every_batch_element(cfg2):
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    q, psi = cfg2
    op = sw.WilsonDirac(q, 0.1)
    got = npy(op.normal(psi))
    ref = O.normal_op(O.fermion_links(q), psi, 0.1)
    err = per_element_rel(got, ref)
    assert err.shape == (4096,) and err.max() < TOL_OP, (err.argmax(), err.max())


def test_cfg2_ddagd_linear_and_hermitian_over_the_batch(cfg2):
    import paper_1512_03812_b200 as sw
    q, psi = cfg2
    op = sw.WilsonDirac(q, 0.1)
    x = torch.as_tensor(psi, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(2)
    y = torch.randn(x.shape, dtype=torch.complex128, device="cuda", generator=g)
    a, b = 0.75 - 0.5j, -1.25 + 2.0j
    Ax, Ay = op.normal(x), op.normal(y)
    lin = op.normal(a * x + b * y) - (a * Ax + b * Ay)
    assert float(lin.abs().max() / Ax.abs().max()) < 1e-13
    # <x, A y> = <A x, y> per chain; <x, A x> real and > 0
    xay = torch.sum(x.conj() * Ay, dim=(1, 2, 3))
    axy = torch.sum(Ax.conj() * y, dim=(1, 2, 3))
    assert float(((xay - axy).abs() / xay.abs()).max()) < 1e-12
    xax = torch.sum(x.conj() * Ax, dim=(1, 2, 3))
    assert float((xax.imag.abs() / xax.real).max()) < 1e-12 and bool((xax.real > 0).all())


def test_cfg2_cg_every_chain_equals_oracle(cfg2):
    """All 4096 per-chain solves: solution <= 1e-12 relative per chain and the
    same iteration count as the oracle's per-chain CG (fermion.py:171-217)."""
    import paper_1512_03812_b200 as sw
    from oracle import parallel as OP
    q, psi = cfg2
    op = sw.WilsonDirac(q, 0.1)
    x, iters, rel = sw.cg_normal(op, psi, 1e-10, stop="per_chain")
    xo, ito = OP.cg_per_chain(q, psi, 0.1, 1e-10)
    its = np.asarray(iters)
    assert its.shape == (4096,) and np.array_equal(its, ito), np.flatnonzero(its != ito)[:8]
    err = per_element_rel(npy(x), xo)
    assert err.max() < TOL_OP, (err.argmax(), err.max())


def test_cfg2_batch_global_cg_true_residual_of_every_chain(cfg2):
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    q, psi = cfg2
    op = sw.WilsonDirac(q, 0.1)
    x, iters, rel = sw.cg_normal(op, psi, 1e-10, stop="batch_global")
    U = O.fermion_links(q)
    rr = true_relres(O, U, 0.1, npy(x), psi)
    assert rr.max() <= 1.0001e-10, rr.max()


def test_cfg3_full_ensemble_update_matches_reference_chains():
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    B, L = 8192, 16
    kw = dict(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
              micro_per_call=2, cg_tol=1e-10)
    cfg, ocfg = sw.HmcConfig(**kw), O.Config(**kw)
    drng = sw.NumpyDeviceRng(seed=2024, n_chains=B)
    q0 = drng.hot_start(sw.LatticeGeom(L, L))
    q1, pend = sw.hmc_update_ensemble_async(q0.clone(), cfg, drng)
    st = pend.resolve()
    q1 = npy(q1)
    # every chain finished with a finite energy change; from a hot start the
    # 4-step schedule accepts ~0.97 of the chains (3 -> 0.86, 5 -> 0.99)
    assert np.isfinite(st.dh).all() and st.accepted.mean() > 0.9
    from oracle import parallel as OP
    chains = sorted(set(range(0, B, 16)) | {1, 4095, 8191})   # 515 chains over the ensemble
    ref = OP.hmc_chains(chains, 2024, kw, n_traj=1)
    q0n = npy(q0)
    for c in chains:
        qs, qo, dh, acc, inv = ref[c]
        assert np.array_equal(qs, q0n[c]), c
        assert abs(st.dh[c] - dh[0]) < 1e-8, c
        assert bool(st.accepted[c]) == bool(acc[0]), c
        assert np.max(np.abs(q1[c] - qo)) < 1e-8, c
    assert int(st.inversions) == int(ref[0][4][0])


def test_cfg4_cluster_cg_every_chain_equals_oracle():
    """All 1024 per-chain 64^2 solves (cluster engine) against the oracle's
    per-chain CG: identical iteration counts, solutions <= 1e-12 per chain,
    and every chain's true residual recomputed by the oracle."""
    import paper_1512_03812_b200 as sw
    from oracle import parallel as OP
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(1024)
    B, L, m0 = 1024, 64, 0.02
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, L))
    b = rng.standard_normal((B, L, L, 2)) + 1j * rng.standard_normal((B, L, L, 2))
    op = sw.WilsonDirac(q, m0)
    x, iters, _ = sw.cg_normal(op, b, 1e-10, stop="per_chain")
    x = npy(x)
    rr = true_relres(O, O.fermion_links(q), m0, x, b)
    assert rr.max() <= 1.0001e-10, rr.max()
    xo, ito = OP.cg_per_chain(q, b, m0, 1e-10)
    its = np.asarray(iters)
    assert np.array_equal(its, ito), np.flatnonzero(its != ito)[:8]
    err = per_element_rel(x, xo)
    assert err.max() < TOL_OP, (err.argmax(), err.max())


@pytest.fixture(scope="module")
def cfg5():
    L = 2048
    rng = np.random.default_rng(5)
    q = rng.uniform(-np.pi, np.pi, (2, L, L))
    psi = rng.standard_normal((L, L, 2)) + 1j * rng.standard_normal((L, L, 2))
    return L, q, psi


@pytest.fixture(scope="module")
def cfg5_one_strip(cfg5):
    """The undecomposed (G = 1) solve of the 2048^2 lattice."""
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    L, q, psi = cfg5
    lat = StripLattice(L, L, strips=1)
    op = DDWilsonDirac(lat, lat.scatter_links(q), 0.05)
    x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
    return npy(lat.gather_spinor(x)), it, rel


@pytest.mark.parametrize("transport,G", [("local", 2), ("p2p", 2), ("local", 8)])
def test_cfg5_decomposed_lattice_full_size(cfg5, cfg5_one_strip, transport, G):
    """2048^2 (configs[4]) on G strips: D^dag D against the oracle on the whole
    lattice; the decomposed CG bit-identical to the one-strip solve (same
    iteration count, same solution bits) and its true residual recomputed
    by the oracle."""
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    from oracle import schwinger_oracle as O
    L, q, psi = cfg5
    lat = StripLattice(L, L, strips=G, transport=transport)
    op = DDWilsonDirac(lat, lat.scatter_links(q), 0.05)
    U = O.fermion_links(q)
    got = npy(lat.gather_spinor(op.normal(lat.scatter_spinor(psi))))
    assert rel_err(got, O.normal_op(U, psi, 0.05)) < TOL_OP
    x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
    x = npy(lat.gather_spinor(x))
    x1, it1, rel1 = cfg5_one_strip
    assert it == it1 and rel == rel1 and np.array_equal(x, x1)
    assert rel <= 1e-10 and it > 0
    rr = true_relres(O, U[None], 0.05, x[None], psi[None])
    assert rr[0] <= 1.0001e-10, rr
