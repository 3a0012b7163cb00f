"""Quenched HMC (HmcConfig.quenched: eta = 0, no pseudofermion draw;
hmc.py:79-80) on every GPU update path, against the reference's own run
(tests/golden/quenched.npz from tests/golden/make_quenched_golden.py): the
unbatched update, measure_dh, the chain ensemble in parity mode and in bench
mode (device NumPy streams), the decomposed lattice and the captured update
graph.  The zero-RHS solves still count their inversions (fermion.py:181-182)."""

from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

L = 12
CASES = [("adapted-nested-fg", 0.25, 2), ("5stage", 0.2, None)]


def npy(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.fixture(scope="module")
def gq():
    return dict(np.load(Path(__file__).resolve().parent / "golden" / "quenched.npz"))


def _cfg(scheme, h, micro):
    import paper_1512_03812_b200 as sw
    return sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=h, scheme=scheme,
                        micro_per_call=micro, cg_tol=1e-10, quenched=True)


@pytest.mark.parametrize("scheme,h,micro", CASES)
def test_quenched_hmc_update_and_measure_dh(gq, scheme, h, micro):
    import paper_1512_03812_b200 as sw
    cfg = _cfg(scheme, h, micro)
    rng = sw.make_rng(5, 0)
    q = sw.hot_start(rng, sw.LatticeGeom(L, L))
    assert np.array_equal(npy(q), gq[f"{scheme}_q0"])
    for k in range(3):
        q, st = sw.hmc_update(q, cfg, rng)
        assert abs(st.dh - gq[f"{scheme}_dh"][k]) < 1e-8
        assert bool(st.accepted) == bool(gq[f"{scheme}_acc"][k])
        assert st.inversions == int(gq[f"{scheme}_inv"][k])
    assert np.max(np.abs(npy(q) - gq[f"{scheme}_q"])) < 1e-8
    m = sw.measure_dh(gq[f"{scheme}_q0"], cfg, sw.make_rng(6, 1), n_samples=8)
    assert np.max(np.abs(np.asarray(m.dh) - gq[f"{scheme}_mdh"])) < 1e-8
    assert m.inversions_per_traj == int(gq[f"{scheme}_minv"])


@pytest.mark.parametrize("scheme,h,micro", CASES)
def test_quenched_ensemble_parity_and_device_streams(gq, scheme, h, micro):
    """Chain 0 of an ensemble is the golden chain (make_rng(5, 0)); chain 1
    is an independent stream checked against the oracle — with host
    generators (parity mode) and with the device NumPy streams."""
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    cfg = _cfg(scheme, h, micro)
    ocfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=h, scheme=scheme,
                    micro_per_call=micro, cg_tol=1e-10, quenched=True)
    rng1 = O.make_rng(5, 1)
    q1 = O.hot_start(rng1, L, L)
    ref1 = []
    for _ in range(3):
        q1, so = O.hmc_update(q1, ocfg, rng1)
        ref1.append((so["dh"], so["accepted"]))
    # parity mode: host generators per chain
    rngs = [sw.make_rng(5, 0), sw.make_rng(5, 1)]
    q = np.stack([npy(sw.hot_start(r, sw.LatticeGeom(L, L))) for r in rngs])
    # bench mode: the same streams walked on the device
    drng = sw.NumpyDeviceRng(seed=5, n_chains=2, stream0=0)
    qd = drng.hot_start(sw.LatticeGeom(L, L))
    assert np.array_equal(npy(qd), q)
    for k in range(3):
        q, st = sw.hmc_update_ensemble(q, cfg, rngs=rngs)
        qd, pend = sw.hmc_update_ensemble_async(qd, cfg, drng)
        sd = pend.resolve()
        for s in (st, sd):
            assert abs(s.dh[0] - gq[f"{scheme}_dh"][k]) < 1e-8
            assert bool(s.accepted[0]) == bool(gq[f"{scheme}_acc"][k])
            assert abs(s.dh[1] - ref1[k][0]) < 1e-8 and bool(s.accepted[1]) == bool(ref1[k][1])
        assert st.inversions == int(gq[f"{scheme}_inv"][k])
    assert np.max(np.abs(npy(q)[0] - gq[f"{scheme}_q"])) < 1e-8
    assert np.max(np.abs(npy(qd)[0] - gq[f"{scheme}_q"])) < 1e-8
    assert np.max(np.abs(npy(q)[1] - q1)) < 1e-8


def test_quenched_update_graph_and_strips(gq):
    """The captured ensemble-update graph on the golden chain, and the
    decomposed lattice."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    scheme, h, micro = CASES[0]
    cfg = _cfg(scheme, h, micro)
    drng = sw.NumpyDeviceRng(seed=5, n_chains=1, stream0=0)
    upd = sw.EnsembleUpdateGraph(drng.hot_start(sw.LatticeGeom(L, L)), cfg, drng)
    for k in range(3):
        upd.step()
        st = upd.stats()
        assert abs(st.dh[0] - gq[f"{scheme}_dh"][k]) < 1e-8
        assert bool(st.accepted[0]) == bool(gq[f"{scheme}_acc"][k])
    assert np.max(np.abs(npy(upd.q)[0] - gq[f"{scheme}_q"])) < 1e-8
    # strips need T % 8 == 0: a 16x16 lattice on 4 strips against the oracle
    # (pinned to the reference's quenched updates by test_oracle_golden.py)
    from oracle import schwinger_oracle as O
    L2 = 16
    kw = dict(L=L2, T=L2, beta=2.0, m0=0.1, tau=1.0, h=h, scheme=scheme, micro_per_call=micro,
              cg_tol=1e-10, quenched=True)
    cfg2, ocfg2 = sw.HmcConfig(**kw), O.Config(**kw)
    lat = StripLattice(L2, L2, strips=4)
    rng, rng_o = sw.make_rng(9, 0), O.make_rng(9, 0)
    qo = O.hot_start(rng_o, L2, L2)
    q_ext = lat.scatter_links(O.hot_start(rng, L2, L2))
    for k in range(3):
        q_ext, st = dd_hmc_update(lat, q_ext, cfg2, rng)
        qo, so = O.hmc_update(qo, ocfg2, rng_o)
        assert abs(st.dh - so["dh"]) < 1e-8
        assert bool(st.accepted) == bool(so["accepted"]) and st.inversions == so["inversions"]
    assert np.max(np.abs(npy(lat.gather_links(q_ext)) - qo)) < 1e-8
