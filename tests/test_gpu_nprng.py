"""The device replica of the reference's NumPy streams (§8(f) row 2):
value-identical draws to make_rng(seed, stream) for every distribution the
HMC path uses, and a device-RNG ensemble that reproduces independent
reference chains trajectory by trajectory."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_standard_normal_stream_is_bit_identical():
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=20240401, n_chains=5, stream0=3)
    got = g.standard_normal((200_000,)).cpu().numpy()    # exercises the ziggurat tail/wedges
    for c in range(5):
        ref = sw.make_rng(20240401, 3 + c).standard_normal(200_000)
        assert np.array_equal(got[c], ref), c
    # the stream continues where it left off
    more = g.standard_normal((7,)).cpu().numpy()
    r = sw.make_rng(20240401, 3)
    r.standard_normal(200_000)
    assert np.array_equal(more[0], r.standard_normal(7))


def test_uniform_random_and_hot_start_are_bit_identical():
    import paper_1512_03812_b200 as sw
    geom = sw.LatticeGeom(6, 10)
    g = sw.NumpyDeviceRng(seed=7, n_chains=3)
    hs = g.hot_start(geom).cpu().numpy()
    u = g.random().cpu().numpy()
    w = g.uniform(-2.5, 4.0, (33,)).cpu().numpy()
    for c in range(3):
        r = sw.make_rng(7, c)
        assert np.array_equal(hs[c], r.uniform(-np.pi, np.pi, size=(2, 6, 10)))
        assert u[c] == r.random()
        assert np.array_equal(w[c], r.uniform(-2.5, 4.0, size=33))


def test_heatbath_draws_match_reference_order():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.fermion import draw_phi
    geom = sw.LatticeGeom(8, 4)
    g = sw.NumpyDeviceRng(seed=11, n_chains=4)
    p, phi = g.heatbath(geom)
    for c in range(4):
        r = sw.make_rng(11, c)
        assert np.array_equal(p[c].cpu().numpy(), r.standard_normal((2, 8, 4)))
        assert np.array_equal(phi[c].cpu().numpy(), draw_phi(r, 8, 4))


def test_metropolis_draws_only_uphill():
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=3, n_chains=4)
    dh = torch.tensor([-0.5, 0.7, 0.0, float("nan")], dtype=torch.float64, device="cuda")
    acc = g.metropolis(dh).cpu().numpy()
    follow = g.random().cpu().numpy()
    for c, d in enumerate([-0.5, 0.7, 0.0]):
        r = sw.make_rng(3, c)
        want = sw.metropolis(d, r)
        assert acc[c] == int(want)
        assert follow[c] == r.random()      # exactly one draw consumed iff dH > 0
    assert acc[3] == -1


def test_device_stream_ensemble_matches_reference_chains():
    """Hot start + 3 trajectories per chain on device streams == the same
    chains run by the CPU oracle with make_rng(seed, c): dH <= 1e-8, same
    accept sequence."""
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    B, L = 3, 8
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    ocfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                    micro_per_call=2, cg_tol=1e-10)
    g = sw.NumpyDeviceRng(seed=99, n_chains=B)
    q = g.hot_start(sw.LatticeGeom(L, L))
    rngs = [O.make_rng(99, c) for c in range(B)]
    qo = np.stack([O.hot_start(r, L, L) for r in rngs])
    assert np.array_equal(q.cpu().numpy(), qo)
    for _ in range(3):
        q, st = sw.hmc_update_ensemble(q, cfg, device_rng=g)
        qo, so = O.ensemble_update(qo, ocfg, rngs)
        assert np.max(np.abs(st.dh - np.array([s["dh"] for s in so]))) < 1e-8
        assert np.array_equal(st.accepted, np.array([s["accepted"] for s in so]))
    assert np.max(np.abs(q.cpu().numpy() - qo)) < 1e-8
