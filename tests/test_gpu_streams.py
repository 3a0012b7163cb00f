"""Concurrent sub-ensembles: each torch stream gets its own library context
(workspace, graph cache, poll flag), so ensembles issued on different streams
with hmc_update_ensemble_async give bit-identical results to one batch."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_two_streams_match_one_batch():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import _lib
    L, B = 8, 6
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    geom = sw.LatticeGeom(L, L)
    g = sw.NumpyDeviceRng(seed=31, n_chains=B)
    q = g.hot_start(geom)
    q1, st1 = sw.hmc_update_ensemble(q, cfg, device_rng=g)
    q1, st1b = sw.hmc_update_ensemble(q1, cfg, device_rng=g)

    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    parts = [(0, 4), (4, 6)]
    rngs, qs = [], []
    for (a, b), s in zip(parts, streams):
        s.wait_stream(main)
        with torch.cuda.stream(s):
            r = sw.NumpyDeviceRng(seed=31, n_chains=b - a, stream0=a)
            rngs.append(r)
            qs.append(r.hot_start(geom))
    dhs = [[], []]
    for _ in range(2):
        pend = []
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                qs[i], p = sw.hmc_update_ensemble_async(qs[i], cfg, rngs[i])
                pend.append(p)
        for i, p in enumerate(pend):
            dhs[i].append(p.resolve().dh)
    for s in streams:
        main.wait_stream(s)
    assert np.array_equal(np.concatenate([dhs[0][0], dhs[1][0]]), st1.dh)
    assert np.array_equal(np.concatenate([dhs[0][1], dhs[1][1]]), st1b.dh)
    assert torch.equal(torch.cat(qs), q1)
    keys = [k for k in _lib._contexts if k[0] == torch.cuda.current_device()]
    assert len(keys) >= 3   # default stream + the two side streams


@pytest.mark.parametrize("L", [8, 16])
def test_captured_update_graph_matches_eager(L):
    """EnsembleUpdateGraph (one CUDA-graph replay per HMC update) gives the
    values of eager hmc_update_ensemble on the same device streams."""
    import paper_1512_03812_b200 as sw
    B = 4
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    geom = sw.LatticeGeom(L, L)
    ge = sw.NumpyDeviceRng(seed=77, n_chains=B)
    qe = ge.hot_start(geom)
    gg = sw.NumpyDeviceRng(seed=77, n_chains=B)
    qg = gg.hot_start(geom)
    upd = sw.EnsembleUpdateGraph(qg, cfg, gg)
    assert torch.equal(gg.state, ge.state)      # capture consumed no draws
    for _ in range(3):
        qe, st = sw.hmc_update_ensemble(qe, cfg, device_rng=ge)
        upd.step()
        sg = upd.stats()
        assert np.array_equal(sg.dh, st.dh)
        assert np.array_equal(sg.accepted, st.accepted)
        assert sg.inversions == st.inversions
    assert torch.equal(upd.q, qe)
    assert torch.equal(gg.state, ge.state)
