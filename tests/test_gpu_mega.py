"""The trajectory megakernel (csrc/mega.cu) against the
kernel-per-map path it replaces and against the oracle's hmc_update."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cfg(sw, **kw):
    base = dict(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                micro_per_call=2, cg_tol=1e-10)
    base.update(kw)
    return sw.HmcConfig(**base)


def _run(sw, cfg, B, mega, updates=2, seed=11):
    sw.hmc.USE_MEGA = mega
    try:
        d = sw.NumpyDeviceRng(seed=seed, n_chains=B)
        q = d.hot_start(sw.LatticeGeom(cfg.L, cfg.T))
        out = []
        for _ in range(updates):
            q, st = sw.hmc_update_ensemble(q, cfg, device_rng=d)
            out.append(st)
        return q.cpu().numpy(), out
    finally:
        sw.hmc.USE_MEGA = False


@pytest.mark.parametrize("h,micro", [(0.25, 2), (0.2, 3)])
def test_megakernel_equals_kernel_per_map_path(h, micro):
    import paper_1512_03812_b200 as sw
    cfg = _cfg(sw, h=h, micro_per_call=micro)
    qa, sa = _run(sw, cfg, 96, True)   # megakernel
    qb, sb = _run(sw, cfg, 96, False)
    for x, y in zip(sa, sb):
        assert np.max(np.abs(x.dh - y.dh)) < 1e-11
        assert np.array_equal(x.accepted, y.accepted)
        assert x.inversions == y.inversions and x.n_steps == y.n_steps
    assert np.max(np.abs(qa - qb)) < 1e-12


def test_megakernel_matches_reference_chains():
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    B = 4
    kw = dict(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
              micro_per_call=2, cg_tol=1e-10)
    cfg, ocfg = sw.HmcConfig(**kw), O.Config(**kw)
    q0, rngs_o = O.ensemble_hot_start(ocfg, B, seed=3)
    _, rngs_g = O.ensemble_hot_start(ocfg, B, seed=3)
    qo, qg = q0, sw.lattice.as_links(q0)
    sw.hmc.USE_MEGA = True
    try:
        assert sw.hmc._mega_eligible(cfg, True)
        for _ in range(3):
            qo, so = O.ensemble_update(qo, ocfg, rngs_o)
            qg, sg = sw.hmc_update_ensemble(qg, cfg, rngs=rngs_g)
            assert np.max(np.abs(sg.dh - np.array([s["dh"] for s in so]))) < 1e-8
            assert np.array_equal(sg.accepted, np.array([s["accepted"] for s in so]))
            assert sg.inversions == so[0]["inversions"]
    finally:
        sw.hmc.USE_MEGA = False
    assert np.max(np.abs(qg.cpu().numpy() - qo)) < 1e-8


def test_megakernel_in_captured_update_graph():
    """EnsembleUpdateGraph replays the megakernel path; values == eager."""
    import paper_1512_03812_b200 as sw
    cfg = _cfg(sw)
    B = 8
    d1 = sw.NumpyDeviceRng(seed=5, n_chains=B)
    d2 = sw.NumpyDeviceRng(seed=5, n_chains=B)
    geom = sw.LatticeGeom(16, 16)
    q1, q2 = d1.hot_start(geom), d2.hot_start(geom)
    sw.hmc.USE_MEGA = True
    try:
        upd = sw.EnsembleUpdateGraph(q2, cfg, d2)
        for _ in range(3):
            q1, s1 = sw.hmc_update_ensemble(q1, cfg, device_rng=d1)
            upd.step()
        torch.cuda.synchronize()
    finally:
        sw.hmc.USE_MEGA = False
    assert torch.equal(q1, upd.q)
