"""Parity of the sm_100a path (through the C-ABI) with the reference.

Inputs and expected outputs come from tests/golden/*.npz, written by running
the reference itself (tests/golden/make_golden.py).  Tolerances (north_star,
BASELINE.json): D^dag D, CG solutions and forces <= 1e-12 relative
(complex128); dH of fixed-seed trajectories <= 1e-8 absolute with the
identical accept/reject sequence; CG iteration counts identical.
Real-arithmetic link updates (drift, wrap) are bit-exact.
"""

import numpy as np
import pytest
import torch

from conftest import rel_err

pytestmark = pytest.mark.gpu

TOL_OP = 1e-12       # operator / solution / force relative tolerance
TOL_DH = 1e-8        # absolute dH tolerance


@pytest.fixture(scope="module")
def sw():
    import paper_1512_03812_b200 as sw
    return sw


def npy(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


STENCIL_CASES = ("s4", "s16", "b6x10", "s2", "s3x5", "s32", "ap8")


@pytest.mark.parametrize("case", STENCIL_CASES)
def test_stencil_matches_reference(sw, golden, case):
    g = golden("stencil")
    bc = "antiperiodic" if case == "ap8" else "periodic"
    op = sw.WilsonDirac(g[f"{case}_q"], float(g[f"{case}_m0"]), fermion_bc=bc)
    psi = g[f"{case}_psi"]
    assert rel_err(npy(op.apply(psi)), g[f"{case}_D"]) < TOL_OP
    assert rel_err(npy(op.apply_dag(psi)), g[f"{case}_Ddag"]) < TOL_OP
    assert rel_err(npy(op.normal(psi)), g[f"{case}_DdD"]) < TOL_OP


@pytest.mark.parametrize("B,L,T", [(3, 32, 16), (2, 8, 64), (5, 48, 32), (1, 16, 32)])
def test_tma_stencil_shapes_match_oracle(sw, B, L, T):
    """Shapes served by the TMA-pipelined D^dag D (whole time rows) and by the
    streaming CG's TMA stencil pass, against the oracle."""
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(L * T + B)
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, T))
    psi = rng.standard_normal((B, L, T, 2)) + 1j * rng.standard_normal((B, L, T, 2))
    op = sw.WilsonDirac(q, 0.1)
    ref = O.normal_op(O.fermion_links(q), psi, 0.1)
    assert rel_err(npy(op.normal(psi)), ref) < TOL_OP
    x, it, _ = sw.cg_normal(op, psi, 1e-10, stop="batch_global")
    xo, ito, _ = O.cg_normal(O.fermion_links(q), 0.1, psi, 1e-10, stop="batch_global")
    assert it == ito
    assert rel_err(npy(x), xo) < TOL_OP


def test_reference_stencil_kats(sw):
    """Free constant mode and point-source stencil (reference test_fermion.py:25-48)."""
    q = np.zeros((2, 4, 4))
    op = sw.WilsonDirac(q, -0.231367)
    psi = np.ones((4, 4, 2), dtype=np.complex128)
    psi[..., 1] = 0.3 - 0.2j
    assert np.allclose(npy(op.apply(psi)), -0.231367 * psi, atol=1e-14)
    assert np.allclose(npy(op.apply_dag(psi)), -0.231367 * psi, atol=1e-14)
    op = sw.WilsonDirac(q, 0.0)
    psi = np.zeros((4, 4, 2), dtype=np.complex128)
    psi[1, 1, 0] = 1.0
    out = npy(op.apply(psi))
    assert np.isclose(out[1, 1, 0], 2.0)
    assert np.isclose(out[0, 1, 0], -0.5) and np.isclose(out[0, 1, 1], 0.5)
    assert np.isclose(out[2, 1, 0], -0.5) and np.isclose(out[2, 1, 1], -0.5)
    assert np.isclose(out[1, 0, 0], -0.5) and np.isclose(out[1, 0, 1], 0.5j)
    assert np.isclose(out[1, 2, 0], -0.5) and np.isclose(out[1, 2, 1], -0.5j)
    mask = np.ones((4, 4), dtype=bool)
    mask[[1, 2, 0, 1, 1], [1, 1, 1, 2, 0]] = False
    assert np.all(out[mask] == 0.0)


def test_operator_identities(sw):
    """Adjoint and gamma5-hermiticity (reference test_fermion.py:59-71)."""
    rng = np.random.default_rng(5)
    q = 0.3 * rng.standard_normal((2, 6, 4))
    op = sw.WilsonDirac(q, -0.231367)
    phi = rng.standard_normal((6, 4, 2)) + 1j * rng.standard_normal((6, 4, 2))
    psi = rng.standard_normal((6, 4, 2)) + 1j * rng.standard_normal((6, 4, 2))
    lhs = complex(sw.spinor_dot(phi, op.apply(psi)).item())
    rhs = complex(sw.spinor_dot(op.apply_dag(phi), psi).item())
    assert abs(lhs - rhs) < 1e-12 * abs(lhs)
    s3 = np.array([1.0, -1.0])
    assert np.max(np.abs(s3 * npy(op.apply(s3 * psi)) - npy(op.apply_dag(psi)))) < 1e-13


@pytest.mark.parametrize("tag,m0,tol", [("a", 0.1, 1e-10), ("d", 0.1, 1e-10), ("e", -0.231367, 1e-12)])
@pytest.mark.parametrize("stop", ["batch_global", "per_chain"])
def test_cg_single_chain_matches_reference(sw, golden, tag, m0, tol, stop):
    g = golden("cg")
    op = sw.WilsonDirac(g[f"{tag}_q"], m0)
    x, it, rel = sw.cg_normal(op, g[f"{tag}_b"], tol, stop=stop)
    assert it == int(g[f"{tag}_it"])
    assert rel_err(npy(x), g[f"{tag}_x"]) < TOL_OP
    assert rel <= tol


def test_cg_warm_start(sw, golden):
    g = golden("cg")
    op = sw.WilsonDirac(g["c_q"], -0.231367)
    x, it, _ = sw.cg_normal(op, g["c_b"], 1e-12, x0=g["c_x0"])
    assert it == int(g["c_it"])
    assert rel_err(npy(x), g["c_x"]) < TOL_OP


def test_cg_batch_global_matches_reference_batched(sw, golden):
    g = golden("cg")
    op = sw.WilsonDirac(g["b_q"], 0.05)
    x, it, _ = sw.cg_normal(op, g["b_b"], 1e-10, stop="batch_global")
    assert it == int(g["b_it_global"])
    assert rel_err(npy(x), g["b_x_global"]) < TOL_OP


def test_cg_per_chain_matches_unbatched_reference(sw, golden):
    g = golden("cg")
    op = sw.WilsonDirac(g["b_q"], 0.05)
    x, its, _ = sw.cg_normal(op, g["b_b"], 1e-10, stop="per_chain")
    assert np.array_equal(its, g["b_it_chain"])
    for c in range(4):
        assert rel_err(npy(x[c]), g["b_x_chain"][c]) < TOL_OP


def test_cg_zero_rhs_and_counter(sw):
    op = sw.WilsonDirac(0.3 * np.random.default_rng(1).standard_normal((2, 4, 4)), -0.231367)
    counter = sw.InversionCounter()
    x, rep = sw.solve_normal(op, np.zeros((4, 4, 2), complex), 1e-12, counter=counter)
    assert np.all(npy(x) == 0.0) and rep.iterations == 0
    assert counter.count == 2
    b = np.zeros((3, 4, 4, 2), complex)
    b[1] = 1.0
    opb = sw.WilsonDirac(np.zeros((3, 2, 4, 4)), 0.1)
    x, its, _ = sw.cg_normal(opb, b, 1e-12, stop="per_chain")
    assert its[0] == 0 and its[2] == 0 and its[1] > 0
    x, it, _ = sw.cg_normal(opb, np.zeros_like(b), 1e-12, stop="batch_global")
    assert it == 0 and np.all(npy(x) == 0)


@pytest.mark.parametrize("stop", ["batch_global", "per_chain"])
def test_cg_cap_raises(sw, golden, stop):
    g = golden("cg")
    op = sw.WilsonDirac(g["a_q"], 0.1)
    with pytest.raises(sw.SolverError) as err:
        sw.cg_normal(op, g["a_b"], 1e-10, maxiter=3, stop=stop)
    assert err.value.best_residual > 0


def test_cg_streaming_engine_matches_oracle(sw):
    """V > 2048 forces the HBM-streaming engine in per-chain mode; compare
    with the oracle's per-chain CG (iteration counts identical)."""
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(11)
    q = rng.uniform(-np.pi, np.pi, (2, 2, 48, 48))
    b = rng.standard_normal((2, 48, 48, 2)) + 1j * rng.standard_normal((2, 48, 48, 2))
    op = sw.WilsonDirac(q, 0.1)
    x, its, _ = sw.cg_normal(op, b, 1e-10, stop="per_chain")
    xo, itso, _ = O.cg_normal(O.fermion_links(q), 0.1, b, 1e-10, stop="per_chain")
    assert np.array_equal(its, itso)
    assert rel_err(npy(x), xo) < TOL_OP


@pytest.mark.parametrize("m0", [0.1, 0.02])
def test_cg_cluster_engine_matches_oracle(sw, m0):
    """64^2 per-chain solves run on the cluster-resident engine (8 CTAs per
    chain, DSMEM faces): iteration counts identical to the oracle's per-chain
    CG, x within 1e-12; a zero right-hand side and a warm start included."""
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(64)
    q = rng.uniform(-np.pi, np.pi, (3, 2, 64, 64))
    b = rng.standard_normal((3, 64, 64, 2)) + 1j * rng.standard_normal((3, 64, 64, 2))
    b[1] = 0.0
    op = sw.WilsonDirac(q, m0)
    x, its, _ = sw.cg_normal(op, b, 1e-10, stop="per_chain")
    xo, itso, _ = O.cg_normal(O.fermion_links(q), m0, b, 1e-10, stop="per_chain")
    assert np.array_equal(its, itso) and its[1] == 0 and its.max() > 50
    assert rel_err(npy(x), xo) < TOL_OP
    x0 = xo + 1e-3 * rng.standard_normal(xo.shape)
    xw, itw, _ = sw.cg_normal(op, b, 1e-10, x0=x0, stop="per_chain")
    xwo, itwo, _ = O.cg_normal(O.fermion_links(q), m0, b, 1e-10, x0=x0, stop="per_chain")
    assert np.array_equal(itw, itwo)
    assert rel_err(npy(xw), xwo) < TOL_OP
    with pytest.raises(sw.SolverError):
        sw.cg_normal(op, b, 1e-10, maxiter=5, stop="per_chain")


@pytest.mark.parametrize("tag", ["u", "b"])
def test_force_pieces_match_reference(sw, golden, tag):
    """link_bilinears (both directions), oriented_plaquettes, plaquette_stencil
    against the reference's own outputs (tests/golden/pieces.npz)."""
    g = golden("pieces")
    op = sw.WilsonDirac(g[f"{tag}_q"], 0.1)
    for mu in (0, 1):
        A, B = sw.link_bilinears(op, mu, g[f"{tag}_a"], g[f"{tag}_b"])
        assert A.shape == g[f"{tag}_A{mu}"].shape
        assert rel_err(npy(A), g[f"{tag}_A{mu}"]) < TOL_OP
        assert rel_err(npy(B), g[f"{tag}_B{mu}"]) < TOL_OP
    P = sw.oriented_plaquettes(g[f"{tag}_q"])
    st = sw.plaquette_stencil(g[f"{tag}_q"])
    assert P.shape == g[f"{tag}_P"].shape and st.shape == g[f"{tag}_stencil"].shape
    assert rel_err(npy(P), g[f"{tag}_P"]) < TOL_OP
    assert rel_err(npy(st), g[f"{tag}_stencil"]) < TOL_OP


@pytest.mark.parametrize("tag", ["u", "b"])
def test_forces_match_reference(sw, golden, tag):
    g = golden("forces")
    q, eta, p = g[f"{tag}_q"], g[f"{tag}_eta"], g[f"{tag}_p"]
    beta, m0, tol = 2.0, 0.1, 1e-12
    op = sw.WilsonDirac(q, m0)
    chi, xi, _ = sw.chi_xi(op, eta, tol)
    assert rel_err(npy(chi), g[f"{tag}_chi"]) < TOL_OP
    assert rel_err(npy(xi), g[f"{tag}_xi"]) < TOL_OP
    assert rel_err(npy(sw.fermion_force(op, chi, xi)), g[f"{tag}_f"]) < TOL_OP
    from paper_1512_03812_b200 import fermion as F
    b1, b2 = F.weighted_w_sums(op, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"])
    assert rel_err(npy(b1), g[f"{tag}_b1"]) < TOL_OP
    assert rel_err(npy(b2), g[f"{tag}_b2"]) < TOL_OP
    # the Z pair and the FG contractions at the north_star bar (measured on B200,
    # tools/parity_errors.py: <= 2.4e-13 for every piece of both cases)
    z1, z2 = F.z_pair(op, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"], tol)
    assert rel_err(npy(z1), g[f"{tag}_z1"]) < TOL_OP
    assert rel_err(npy(z2), g[f"{tag}_z2"]) < TOL_OP
    fgff = F.fg_fermion_hessian_dot(op, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_f"], tol)
    assert rel_err(npy(fgff), g[f"{tag}_fgff"]) < TOL_OP
    fggf = F.fg_fermion_hessian_dot(op, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_g"], tol)
    assert rel_err(npy(fggf), g[f"{tag}_fggf"]) < TOL_OP
    assert rel_err(npy(sw.gauge_force(q, beta)), g[f"{tag}_g"]) < 1e-14
    from paper_1512_03812_b200 import gauge as G
    assert np.array_equal(npy(G.plaq_angles(q)), g[f"{tag}_plaq"])
    assert rel_err(npy(sw.fg_gauge_gauge(q, beta)), g[f"{tag}_fggg"]) < 1e-14
    assert rel_err(npy(sw.gauge_hessian_dot(q, beta, g[f"{tag}_f"])), g[f"{tag}_ghd"]) < 1e-14
    assert rel_err(npy(sw.gauge_action(q, beta)), g[f"{tag}_SG"]) < 1e-14
    assert rel_err(npy(sw.avg_plaquette(q)), g[f"{tag}_avgP"]) < 1e-14
    assert rel_err(npy(sw.kinetic_energy(p)), g[f"{tag}_kin"]) < 1e-14
    assert np.array_equal(npy(sw.rotate_links(q, p, 0.37)), g[f"{tag}_drift"])
    assert np.array_equal(npy(sw.wrap_angles(4.0 * q)), g[f"{tag}_wrap"])
    assert rel_err(npy(sw.fermion_action(op, eta, tol)), g[f"{tag}_SF"]) < TOL_OP


def test_measure_dh_matches_reference(sw, golden):
    g = golden("measure")
    for k, scheme in enumerate(("adapted-nested-fg", "5stage-fg", "leapfrog")):
        cfg = sw.HmcConfig(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                           micro_per_call=2 if scheme.startswith("adapted") else None,
                           cg_tol=1e-12, seed=11)
        rng = sw.make_rng(11, k)
        q0 = 0.4 * rng.standard_normal((2, 6, 6))
        m = sw.measure_dh(q0, cfg, rng, n_samples=5)
        assert m.inversions_per_traj == int(g[f"m{k}_inv"])
        assert np.max(np.abs(m.dh - g[f"m{k}_dh"])) < TOL_DH


def test_all_schemes_match_reference(sw, golden):
    g = golden("traj")
    for k, scheme in enumerate(sw.SCHEME_IDS):
        cfg = sw.HmcConfig(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                           micro_per_call=2 if scheme in ("nested-leapfrog", "nested-5stage",
                                                          "nested-fg", "adapted-nested-fg") else None,
                           cg_tol=1e-12, seed=3)
        rng = sw.make_rng(3, k)
        q = 0.4 * rng.standard_normal((2, 6, 6))
        for t in range(2):
            q, s = sw.hmc_update(q, cfg, rng)
            assert abs(s.dh - g[f"sch{k}_dh"][t]) < TOL_DH, scheme
            assert s.accepted == bool(g[f"sch{k}_acc"][t]), scheme
            assert s.inversions == int(g[f"sch{k}_inv"][t]), scheme
        assert np.max(np.abs(npy(q) - g[f"sch{k}_qlast"])) < TOL_DH, scheme


@pytest.mark.parametrize("tag,h,n,bc", [("cfg1", 0.2, 20, "periodic"),
                                        ("cfg1h3", 1.0 / 3.0, 20, "periodic"),
                                        ("cfg1ap", 0.2, 5, "antiperiodic")])
def test_cfg1_trajectories_match_reference(sw, golden, tag, h, n, bc):
    """BASELINE configs[0] (16x16, beta 2, m0 0.1, adapted nested FG, 5x2 steps,
    tol 1e-10) and its rejecting h=1/3 twin: dH <= 1e-8, same accept sequence."""
    g = golden("traj")
    cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=h, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10, seed=0, fermion_bc=bc)
    rng = sw.make_rng(0, 0)
    q = sw.hot_start(rng, sw.LatticeGeom(16, 16))
    assert np.array_equal(npy(q), g[f"{tag}_q0"])
    for t in range(n):
        q, s = sw.hmc_update(q, cfg, rng)
        assert abs(s.dh - g[f"{tag}_dh"][t]) < TOL_DH, t
        assert s.accepted == bool(g[f"{tag}_acc"][t]), t
        assert s.inversions == int(g[f"{tag}_inv"][t])
    assert np.max(np.abs(npy(q) - g[f"{tag}_qlast"])) < TOL_DH


def test_ensemble_matches_independent_reference_chains(sw):
    """hmc_update_ensemble over B chains == B unbatched oracle hmc_update calls."""
    from oracle import schwinger_oracle as O
    B, L = 4, 8
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    ocfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=0.25, scheme="adapted-nested-fg",
                    micro_per_call=2, cg_tol=1e-10)
    q0, rngs_o = O.ensemble_hot_start(ocfg, B, seed=7)
    _, rngs_g = O.ensemble_hot_start(ocfg, B, seed=7)
    qo, qg = q0, sw.lattice.as_links(q0)
    for _ in range(3):
        qo, so = O.ensemble_update(qo, ocfg, rngs_o)
        qg, sg = sw.hmc_update_ensemble(qg, cfg, rngs=rngs_g)
        assert np.max(np.abs(sg.dh - np.array([s["dh"] for s in so]))) < TOL_DH
        assert np.array_equal(sg.accepted, np.array([s["accepted"] for s in so]))
        assert sg.inversions == so[0]["inversions"]
    assert np.max(np.abs(npy(qg) - qo)) < TOL_DH


def test_solve_reuse_is_bit_identical(sw):
    """Reusing chi/xi across FSAL kicks and the Hamiltonian changes nothing."""
    cfg = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.2, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    out = []
    for reuse in (True, False):
        rng = sw.make_rng(0, 0)
        q = sw.hot_start(rng, sw.LatticeGeom(16, 16))
        trace = []
        for _ in range(2):
            q, s = sw.hmc_update(q, cfg, rng, reuse_solves=reuse)
            trace.append((s.dh, s.accepted, s.inversions))
        out.append((trace, npy(q)))
    assert out[0][0] == out[1][0]
    assert np.array_equal(out[0][1], out[1][1])


def test_runs_are_bit_deterministic(sw):
    """Fixed-order reductions: two identical runs give identical traces
    (reference test_hmc.py:115-130)."""
    cfg = sw.HmcConfig(L=8, T=8, beta=1.0, m0=0.1, tau=1.0, h=0.1, scheme="leapfrog", cg_tol=1e-12)

    def run():
        rng = sw.make_rng(5, 2)
        q = 0.3 * rng.standard_normal((2, 8, 8))
        trace = []
        for _ in range(3):
            q, s = sw.hmc_update(q, cfg, rng)
            trace.append((s.dh, s.accepted, s.inversions))
        return trace, npy(q)

    a, b = run(), run()
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_reject_returns_original_object(sw):
    cfg = sw.HmcConfig(L=4, T=4, beta=1.0, m0=-0.231367, tau=0.9, h=0.45, scheme="leapfrog",
                       cg_tol=1e-12, seed=5)
    rng = sw.make_rng(12, 0)
    q = 0.3 * sw.make_rng(20240401, 0).standard_normal((2, 4, 4))
    for _ in range(20):
        q_new, s = sw.hmc_update(q, cfg, rng)
        if not s.accepted:
            assert q_new is q
            return
        q = q_new
    pytest.fail("no rejection at a violently unstable step size")


def test_wrap_angles_bit_exact_stress(sw):
    """The device floored remainder (FMA with a corrected quotient instead of
    the library fmod loop) is bit-identical to NumPy's on a million angles,
    including exact multiples of 2pi, boundary neighbours and large values."""
    from oracle import schwinger_oracle as O
    rng = np.random.default_rng(2)
    two_pi = 2.0 * np.pi
    k = rng.integers(-40, 40, 200_000).astype(np.float64)
    edge = np.concatenate([k * two_pi - np.pi, np.nextafter(k * two_pi - np.pi, np.inf),
                           np.nextafter(k * two_pi - np.pi, -np.inf)])
    vals = np.concatenate([rng.uniform(-4 * np.pi, 4 * np.pi, 300_000),
                           rng.standard_normal(100_000) * 1e3, rng.standard_normal(50_000) * 1e9,
                           edge, [0.0, -0.0, np.pi, -np.pi, 1e14, -1e14]])
    got = sw.wrap_angles(vals).cpu().numpy()
    want = O.wrap_angles(vals)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


_BASIS_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1512_03812_b200 as sw
from paper_1512_03812_b200 import fermion as F
out = {}
for L, B in ((16, 6), (32, 3), (64, 2)):
    rng = np.random.default_rng(100 + L)
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, L))
    b = rng.standard_normal((B, L, L, 2)) + 1j * rng.standard_normal((B, L, L, 2))
    op = sw.WilsonDirac(q, 0.1)
    x, info = F.cg_solve(op, b, 1e-10, stop="per_chain")
    out[f"x{L}"] = x.cpu().numpy()
    out[f"it{L}"] = info.iters_dev.cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def test_resident_cg_spin_basis_matches_reference_basis(tmp_path):
    """The resident engines solve in the sigma1-diagonal spin basis by default
    (block_stencil.cuh SiteBlockRot); SCH_RESBLK_ROT=0 runs the reference
    basis.  Both must give the same solutions (<= 1e-12 relative, the CG
    tolerance bar) and the same iteration counts on the 16^2 / 32^2 block
    kernels and the 64^2 cluster kernel.  The switch is read once per
    process, so each basis runs in its own interpreter."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for rot in ("0", "1"):
        path = tmp_path / f"rot{rot}.npz"
        env = dict(os.environ, SCH_RESBLK_ROT=rot)
        subprocess.run([sys.executable, "-c", _BASIS_SNIPPET, root, str(path)], check=True, env=env,
                       timeout=300)
        res[rot] = np.load(path)
    for L in (16, 32, 64):
        a, b = res["0"][f"x{L}"], res["1"][f"x{L}"]
        assert rel_err(b, a) <= TOL_OP, (L, rel_err(b, a))
        np.testing.assert_array_equal(res["0"][f"it{L}"], res["1"][f"it{L}"])


def test_thermalize_matches_reference(sw):
    """thermalize (hmc.py:133-155): cold start, 60 leapfrog updates with the
    reference's step annealing (it fires once: 0.1 -> 0.07) at the paper's
    mass on 8x8, against the reference's own run (tests/golden/therm.npz)."""
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "therm.npz")
    cfg = sw.HmcConfig(L=8, T=8, beta=1.0, m0=-0.231367, tau=1.0, h=0.1, cg_tol=1e-10,
                       n_thermalize=60, seed=11)
    q, hist = sw.thermalize(cfg, sw.make_rng(11, 0))
    hist, ref = np.asarray(hist), g["history"]
    # the same accept/reject sequence (a rejection repeats the plaquette) and
    # so the same annealing; the chains agree to rounding at first, and at
    # this light mass the molecular dynamics amplify the rounding-level
    # difference of each trajectory (1e-13 -> ~1e-11 after 5 updates ->
    # ~1e-6 after 60, measured), as between any two float64 implementations
    assert np.array_equal(np.diff(hist) == 0, np.diff(ref) == 0)
    assert np.max(np.abs(hist[:5] - ref[:5])) < 1e-10
    assert np.max(np.abs(hist - ref)) < 1e-4
    assert np.max(np.abs(q.cpu().numpy() - g["q"])) < 1e-3
    from dataclasses import replace
    q5, _ = sw.thermalize(replace(cfg, n_thermalize=5), sw.make_rng(11, 0))
    assert np.max(np.abs(q5.cpu().numpy() - g["q5"])) < 1e-9
