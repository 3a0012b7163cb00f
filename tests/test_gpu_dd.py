"""Domain-decomposed D^dag D and CG (BASELINE configs[4]) against the
single-lattice path and the oracle, with every strip on one GPU (local
transport: the same CG loop, halo rows filled by a copy kernel instead of
NCCL send/recv)."""

import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu


def npy(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("transport", ["local", "p2p"])
@pytest.mark.parametrize("L,T,G", [(64, 32, 4), (32, 128, 2), (48, 16, 6), (16, 8, 8)])
def test_dd_normal_and_cg_match_single_lattice(L, T, G, transport):
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(L + T + G)
    q = rng.uniform(-np.pi, np.pi, (2, L, T))
    psi = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    lat = StripLattice(L, T, strips=G, transport=transport)
    assert (lat.S, lat.Lloc, lat.Lext) == (G, L // G, L // G + 4)
    op = DDWilsonDirac(lat, lat.scatter_links(q), 0.1)
    ref = O.normal_op(O.fermion_links(q), psi, 0.1)
    assert rel_err(npy(lat.gather_spinor(op.normal(lat.scatter_spinor(psi)))), ref) < 1e-12
    x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
    xo, ito, _ = O.cg_normal(O.fermion_links(q), 0.1, psi, 1e-10)
    assert it == ito
    assert rel <= 1e-10
    assert rel_err(npy(lat.gather_spinor(x)), xo) < 1e-12
    # the single-lattice GPU path agrees too
    xs, its, _ = sw.cg_normal(sw.WilsonDirac(q, 0.1), psi, 1e-10)
    assert its == it


@pytest.mark.parametrize("scheme,h,G", [("adapted-nested-fg", 0.25, 4), ("5stage", 0.2, 2),
                                        ("nested-leapfrog", 0.25, 8), ("5stage-fg", 0.25, 2),
                                        ("fg-approx", 0.25, 4), ("11stage", 0.5, 2),
                                        ("nested-fg", 0.25, 4), ("nested-5stage", 0.25, 2),
                                        ("leapfrog", 0.125, 4)])
def test_dd_hmc_update_matches_reference_full_lattice(scheme, h, G):
    """HMC on strips (draws from the full-lattice reference generator) ==
    the oracle's hmc_update on the whole lattice: dH <= 1e-8, same accept
    sequence and inversion count, same final links."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    L = 16
    kw = dict(L=L, T=L, beta=2.0, m0=0.1, tau=1.0 if scheme == "adapted-nested-fg" else 0.5, h=h,
              scheme=scheme, micro_per_call=2 if scheme.startswith(("nested", "adapted")) else None,
              cg_tol=1e-10)
    cfg, ocfg = sw.HmcConfig(**kw), O.Config(**kw)
    lat = StripLattice(L, L, strips=G)
    rng_g, rng_o = O.make_rng(4, 0), O.make_rng(4, 0)
    q0 = O.hot_start(rng_g, L, L)
    assert np.array_equal(q0, O.hot_start(rng_o, L, L))
    q_ext, qo = lat.scatter_links(q0), q0
    for _ in range(2):
        q_ext, s = dd_hmc_update(lat, q_ext, cfg, rng_g)
        qo, so = O.hmc_update(qo, ocfg, rng_o)
        assert abs(s.dh - so["dh"]) < 1e-8
        assert s.accepted == so["accepted"] and s.inversions == so["inversions"]
    assert np.max(np.abs(npy(lat.gather_links(q_ext)) - qo)) < 1e-8


@pytest.mark.parametrize("L,T,G", [(256, 256, 2), (96, 192, 3), (40, 128, 5), (64, 64, 16)])
def test_dd_long_rows_match_oracle_and_are_strip_invariant(L, T, G):
    """Decomposed lattices with several 64-wide t-chunks per row (the
    canonical row partials of dd.cu over more than one chunk, the t-wrap
    between tiles, clipped x tiles): D^dag D vs the oracle, and CG
    solutions / iteration counts / residuals bit-identical to one strip
    (power-of-two strip heights: dd.cu's canonical sums)."""
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(L * T + G)
    q = rng.uniform(-np.pi, np.pi, (2, L, T))
    psi = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    ref = O.normal_op(O.fermion_links(q), psi, 0.1)
    runs = []
    for g in (1, G):
        lat = StripLattice(L, T, strips=g)
        op = DDWilsonDirac(lat, lat.scatter_links(q), 0.1)
        got = npy(lat.gather_spinor(op.normal(lat.scatter_spinor(psi))))
        assert rel_err(got, ref) < 1e-12, g
        x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
        runs.append((npy(lat.gather_spinor(x)), it, rel))
    assert runs[0][1] == runs[1][1] and runs[0][2] == runs[1][2]
    assert np.array_equal(runs[0][0], runs[1][0])
    if L * T <= 96 * 192:
        xo, ito, _ = O.cg_normal(O.fermion_links(q), 0.1, psi, 1e-10)
        assert runs[0][1] == ito and rel_err(runs[0][0], xo) < 1e-12


@pytest.mark.parametrize("transport", ["local", "p2p"])
def test_dd_exchange_fills_halos_from_neighbours(transport):
    from paper_1512_03812_b200.dd import StripLattice
    L, T, G = 24, 8, 3
    lat = StripLattice(L, T, strips=G, transport=transport)
    full = torch.arange(L * T * 4, dtype=torch.float64, device="cuda").reshape(L, T, 2, 2)
    psi = torch.view_as_complex(full.contiguous())
    ext = lat.scatter_spinor(psi)
    want = ext.clone()
    ext[:, :2] = 0
    ext[:, -2:] = 0
    lat.exchange(ext, 1, 4)
    assert torch.equal(ext, want)


def _gathered_cg(L, T, G, transport, q, b, m0, tol, x0=None):
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    lat = StripLattice(L, T, strips=G, transport=transport)
    op = DDWilsonDirac(lat, lat.scatter_links(q), m0)
    x, it, rel = op.cg(lat.scatter_spinor(b), tol,
                       x0_ext=None if x0 is None else lat.scatter_spinor(x0))
    return npy(lat.gather_spinor(x)), it, rel


@pytest.mark.parametrize("transport", ["local", "p2p"])
def test_dd_cg_is_bit_identical_for_every_strip_count(transport):
    """Every global sum is the canonical tree over rows (csrc/dd.cu), so the
    decomposed CG takes the same steps with the same bits for G = 1..16 at
    the reference suite's light mass and tol 1e-12 (conftest: m0 -0.231367),
    cold and warm started."""
    L, T = 64, 64
    rng = np.random.default_rng(64)
    q = 0.3 * rng.standard_normal((2, L, T))
    b = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    x0 = 0.1 * (rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2)))
    for warm in (None, x0):
        ref = _gathered_cg(L, T, 1, "local", q, b, -0.231367, 1e-12, warm)
        for G in (2, 4, 8, 16):
            got = _gathered_cg(L, T, G, transport, q, b, -0.231367, 1e-12, warm)
            assert got[1] == ref[1] and got[2] == ref[2], (G, got[1:], ref[1:])
            assert np.array_equal(got[0], ref[0]), G


def test_dd_hmc_update_is_bit_identical_for_every_strip_count():
    """Whole HMC updates on 1, 2, 4 and 8 strips: the same dH, accept and
    final links to the last bit (halo exchanges are exact copies, and the
    CG's and the Hamiltonian's sums are the strip-count invariant tree)."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    L = 32
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=0.5, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    runs = {}
    for G in (1, 2, 4, 8):
        lat = StripLattice(L, L, strips=G)
        rng = O.make_rng(21, 0)
        q_ext = lat.scatter_links(O.hot_start(rng, L, L))
        trace = []
        for _ in range(2):
            q_ext, s = dd_hmc_update(lat, q_ext, cfg, rng)
            trace.append((s.dh, s.accepted, s.inversions))
        runs[G] = (trace, npy(lat.gather_links(q_ext)))
    for G in (2, 4, 8):
        assert runs[G][0] == runs[1][0], G
        assert np.array_equal(runs[G][1], runs[1][1]), G


def test_dd_hmc_update_device_heatbath_equals_host_draws():
    """The device NumPy-stream generator (one stream, whole lattice drawn on
    the GPU, own rows kept) gives the same updates as the host generator:
    same dH bits, accepts (the device Metropolis uniform included) and links,
    over updates that both accept and reject."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    L, G = 32, 4
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=0.5, h=0.5, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    lat = StripLattice(L, L, strips=G)
    rng_h = O.make_rng(33, 0)
    q0 = O.hot_start(rng_h, L, L)
    rng_d = sw.NumpyDeviceRng(seed=33, n_chains=1, stream0=0)
    assert np.array_equal(npy(rng_d.hot_start(sw.LatticeGeom(L, L))[0]), q0)
    qh = qd = lat.scatter_links(q0)
    for _ in range(4):
        qh, sh = dd_hmc_update(lat, qh, cfg, rng_h)
        qd, sd = dd_hmc_update(lat, qd, cfg, rng_d)
        assert (sd.dh, sd.accepted, sd.inversions) == (sh.dh, sh.accepted, sh.inversions)
        assert torch.equal(qd, qh)
    with pytest.raises(ValueError):
        dd_hmc_update(lat, qd, cfg, sw.NumpyDeviceRng(seed=1, n_chains=2))


def test_dd_cg_zero_rhs_warm_start_and_cap():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    L, T, G = 32, 16, 4
    rng = np.random.default_rng(3)
    q = 0.3 * rng.standard_normal((2, L, T))
    lat = StripLattice(L, T, strips=G)
    op = DDWilsonDirac(lat, lat.scatter_links(q), -0.231367)
    zero = torch.zeros((G, L // G + 4, T, 2), dtype=torch.complex128, device="cuda")
    x, it, _ = op.cg(zero, 1e-12)
    assert it == 0 and torch.count_nonzero(x) == 0
    b = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    x0 = 0.1 * (rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2)))
    x, it, rel = op.cg(lat.scatter_spinor(b), 1e-12, x0_ext=lat.scatter_spinor(x0))
    from oracle import schwinger_oracle as O
    xo, ito, _ = O.cg_normal(O.fermion_links(q), -0.231367, b, 1e-12, x0=x0)
    # light mass, tol 1e-12, 234 iterations: the same stopping iteration as the
    # reference rule and the solution at the north_star bar (measured on B200:
    # 2.2e-14; tools/dd_vs_oracle.py)
    assert it == ito
    assert rel <= 1e-12
    assert rel_err(npy(lat.gather_spinor(x)), xo) < 1e-12
    with pytest.raises(sw.SolverError):
        op.cg(lat.scatter_spinor(b), 1e-12, maxiter=3)


@pytest.mark.parametrize("G", [1, 2, 5])
def test_p2p_mailboxes_over_many_exchanges_and_shapes(G):
    """The peer-memory transport (mailbox slots reused by sequence parity,
    credits returned by the pull kernels) on every strip of one process:
    links (2 planes x 1 word) and spinors (1 x 4) interleaved many times,
    each exchange == the copy-kernel transport's halos."""
    from paper_1512_03812_b200.dd import StripLattice
    L, T = 8 * G, 12
    a = StripLattice(L, T, strips=G, transport="p2p")
    b = StripLattice(L, T, strips=G, transport="local")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(G)
    for k in range(7):
        q = torch.rand((2, L, T), dtype=torch.float64, device="cuda", generator=gen)
        psi = torch.randn((L, T, 2), dtype=torch.complex128, device="cuda", generator=gen)
        for field, planes, words in ((b.scatter_links(q), 2, 1), (b.scatter_spinor(psi), 1, 4)):
            want = field.clone()
            x = field.clone()
            axis = 1 if planes == 1 else 2   # the extended row axis
            x.narrow(axis, 0, 2).zero_()
            x.narrow(axis, a.Lext - 2, 2).zero_()
            y = x.clone()
            a.exchange(x, planes, words)
            b.exchange(y, planes, words)
            assert torch.equal(x, y) and torch.equal(x, want)


def test_p2p_rejects_wide_sites_and_bad_transport():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    lat = StripLattice(16, 8, strips=2, transport="p2p")
    f = torch.zeros((2, 3, lat.Lext, 8, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(Exception):
        lat.exchange(f, 3, 2)
    with pytest.raises(ValueError):
        StripLattice(16, 8, strips=2, transport="nccl")
    with pytest.raises(ValueError):
        StripLattice(16, 8, strips=2, transport="udp")


def test_dd_hmc_update_p2p_transport_matches_reference():
    """One scheme end to end on the peer-memory transport (faces after every
    drift, forces, CG exchanges and sums all through the mailboxes)."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    L, G = 16, 4
    kw = dict(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
              micro_per_call=2, cg_tol=1e-10)
    cfg, ocfg = sw.HmcConfig(**kw), O.Config(**kw)
    lat = StripLattice(L, L, strips=G, transport="p2p")
    rng_g, rng_o = O.make_rng(9, 0), O.make_rng(9, 0)
    q0 = O.hot_start(rng_g, L, L)
    O.hot_start(rng_o, L, L)
    q_ext, qo = lat.scatter_links(q0), q0
    for _ in range(2):
        q_ext, s = dd_hmc_update(lat, q_ext, cfg, rng_g)
        qo, so = O.hmc_update(qo, ocfg, rng_o)
        assert abs(s.dh - so["dh"]) < 1e-8
        assert s.accepted == so["accepted"] and s.inversions == so["inversions"]
    assert np.max(np.abs(npy(lat.gather_links(q_ext)) - qo)) < 1e-8


def test_dd_nccl_transport_on_one_rank_matches_local():
    """The NCCL transport's code path (grouped ncclSend/ncclRecv of the faces
    — here to the rank itself — ncclAllGather of the strip values, the
    host-driven CG loop) on a one-rank process group: D^dag D, CG and a whole
    HMC update bit-identical to the local transport.  (Across GPUs the pool
    cannot run it: one GPU.)"""
    import socket
    import torch.distributed as dist
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        L = 64
        rng = np.random.default_rng(17)
        q = rng.uniform(-np.pi, np.pi, (2, L, L))
        psi = rng.standard_normal((L, L, 2)) + 1j * rng.standard_normal((L, L, 2))
        lat_n = StripLattice(L, L, group=dist.group.WORLD, transport="nccl")
        lat_l = StripLattice(L, L, strips=1)
        assert lat_n.transport == "nccl" and (lat_n.world, lat_n.S) == (1, 1)
        res = []
        for lat in (lat_n, lat_l):
            op = DDWilsonDirac(lat, lat.scatter_links(q), 0.1)
            y = npy(lat.gather_spinor(op.normal(lat.scatter_spinor(psi))))
            x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
            res.append((y, npy(lat.gather_spinor(x)), it, rel))
        assert np.array_equal(res[0][0], res[1][0])
        assert np.array_equal(res[0][1], res[1][1]) and res[0][2:] == res[1][2:]
        cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=0.5, h=0.25, scheme="adapted-nested-fg",
                           micro_per_call=2, cg_tol=1e-10)
        out = []
        for lat in (lat_n, lat_l):
            rng_h = O.make_rng(8, 0)
            q0 = lat.scatter_links(O.hot_start(rng_h, L, L))
            q1, st = dd_hmc_update(lat, q0, cfg, rng_h)
            out.append((npy(lat.gather_links(q1)), st.dh, st.accepted, st.inversions))
        assert np.array_equal(out[0][0], out[1][0]) and out[0][1:] == out[1][1:]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme,G", [("adapted-nested-fg", 4), ("fg-approx", 2)])
def test_dd_hmc_update_antiperiodic_matches_reference(scheme, G):
    """Antiperiodic fermion boundary in time (BASELINE configs[0]; the sign
    of U_t on the last time slice, applied per extended strip — strips cut
    x, so every strip holds whole time rows): HMC updates on strips == the
    oracle's antiperiodic hmc_update on the whole lattice."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.dd import StripLattice
    from paper_1512_03812_b200.dd_hmc import dd_hmc_update
    from oracle import schwinger_oracle as O
    L = 16
    kw = dict(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme=scheme,
              micro_per_call=2 if scheme.startswith(("nested", "adapted")) else None,
              cg_tol=1e-10, fermion_bc="antiperiodic")
    cfg, ocfg = sw.HmcConfig(**kw), O.Config(**kw)
    lat = StripLattice(L, L, strips=G)
    rng_g, rng_o = O.make_rng(12, 0), O.make_rng(12, 0)
    q0 = O.hot_start(rng_g, L, L)
    O.hot_start(rng_o, L, L)
    q_ext, qo = lat.scatter_links(q0), q0
    for _ in range(2):
        q_ext, s = dd_hmc_update(lat, q_ext, cfg, rng_g)
        qo, so = O.hmc_update(qo, ocfg, rng_o)
        assert abs(s.dh - so["dh"]) < 1e-8
        assert s.accepted == so["accepted"] and s.inversions == so["inversions"]
    assert np.max(np.abs(npy(lat.gather_links(q_ext)) - qo)) < 1e-8


_MARCH_SNIPPET = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
out = {}
for L, T, G in [(32, 8, 1), (64, 56, 2), (48, 200, 3), (16, 2048, 2), (256, 96, 4)]:
    rng = np.random.default_rng(L * T + G)
    q = rng.uniform(-np.pi, np.pi, (2, L, T))
    psi = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    lat = StripLattice(L, T, strips=G)
    op = DDWilsonDirac(lat, lat.scatter_links(q), 0.1)
    out[f"n_{L}_{T}"] = lat.gather_spinor(op.normal(lat.scatter_spinor(psi))).cpu().numpy()
    x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
    out[f"x_{L}_{T}"] = lat.gather_spinor(x).cpu().numpy()
    out[f"it_{L}_{T}"] = np.array([it])
np.savez(sys.argv[2], **out)
"""


def test_dd_marching_pass_equals_tile_kernels(tmp_path):
    """The warp-marching stencil pass (csrc/march.cuh, the default) against
    the shared-memory tile kernels (SCH_DD_MARCH=0) on rows shorter than a
    warp's band (T = 8), of whole bands (56), with a clipped last band (200,
    96) and of cfg5's length (2048: 512 row partials per row through the
    coalesced canonical sum): D^dag D to 1e-13, the same CG iteration counts,
    solutions to 1e-12.  The switch is read once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for m in ("0", "1"):
        path = tmp_path / f"march{m}.npz"
        env = dict(os.environ, SCH_DD_MARCH=m)
        subprocess.run([sys.executable, "-c", _MARCH_SNIPPET, root, str(path)], check=True, env=env,
                       timeout=600)
        res[m] = np.load(path)
    for k in res["0"].files:
        a, b = res["0"][k], res["1"][k]
        if k.startswith("it_"):
            np.testing.assert_array_equal(a, b, err_msg=k)
        else:
            assert rel_err(b, a) < (1e-13 if k.startswith("n_") else 1e-12), (k, rel_err(b, a))


def test_dd_marching_pass_cfg5_rows_match_oracle():
    """Rows of cfg5's length on a short lattice (16 x 2048, two strips)
    against the oracle: D^dag D to 1e-12, CG iteration count and solution."""
    from paper_1512_03812_b200.dd import DDWilsonDirac, StripLattice
    from oracle import schwinger_oracle as O
    L, T = 16, 2048
    rng = np.random.default_rng(2048)
    q = rng.uniform(-np.pi, np.pi, (2, L, T))
    psi = rng.standard_normal((L, T, 2)) + 1j * rng.standard_normal((L, T, 2))
    U = O.fermion_links(q)
    runs = []
    for G in (1, 2):
        lat = StripLattice(L, T, strips=G)
        op = DDWilsonDirac(lat, lat.scatter_links(q), 0.1)
        got = npy(lat.gather_spinor(op.normal(lat.scatter_spinor(psi))))
        assert rel_err(got, O.normal_op(U, psi, 0.1)) < 1e-12
        x, it, rel = op.cg(lat.scatter_spinor(psi), 1e-10)
        runs.append((npy(lat.gather_spinor(x)), it, rel))
    assert runs[0][1:] == runs[1][1:] and np.array_equal(runs[0][0], runs[1][0])
    xo, ito, _ = O.cg_normal(U, 0.1, psi, 1e-10)
    assert runs[0][1] == ito and rel_err(runs[0][0], xo) < 1e-12
