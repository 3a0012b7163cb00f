"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz,
produced by tests/golden/make_golden.py from /root/reference).  CPU only."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import schwinger_oracle as O

STENCIL_CASES = ("s4", "s16", "b6x10", "s2", "s3x5", "s32")


@pytest.mark.parametrize("case", STENCIL_CASES + ("ap8",))
def test_oracle_stencil_matches_reference(golden, case):
    g = golden("stencil")
    bc = "antiperiodic" if case == "ap8" else "periodic"
    U = O.fermion_links(g[f"{case}_q"], bc)
    m0, psi = float(g[f"{case}_m0"]), g[f"{case}_psi"]
    assert rel_err(O.dirac(U, psi, m0), g[f"{case}_D"]) < 1e-14
    assert rel_err(O.dirac(U, psi, m0, dagger=True), g[f"{case}_Ddag"]) < 1e-14
    assert rel_err(O.normal_op(U, psi, m0), g[f"{case}_DdD"]) < 1e-14


def test_oracle_cg_single_chain(golden):
    g = golden("cg")
    for tag, m0, tol in (("a", 0.1, 1e-10), ("d", 0.1, 1e-10), ("e", -0.231367, 1e-12)):
        U = O.fermion_links(g[f"{tag}_q"])
        for stop in ("batch_global", "per_chain"):
            x, it, _ = O.cg_normal(U, m0, g[f"{tag}_b"], tol, stop=stop)
            assert int(np.max(it)) == int(g[f"{tag}_it"]), (tag, stop)
            assert rel_err(x, g[f"{tag}_x"]) < 1e-12


def test_oracle_cg_warm_start(golden):
    g = golden("cg")
    U = O.fermion_links(g["c_q"])
    x, it, _ = O.cg_normal(U, -0.231367, g["c_b"], 1e-12, x0=g["c_x0"])
    assert it == int(g["c_it"])
    assert rel_err(x, g["c_x"]) < 1e-12


def test_oracle_cg_batch_modes(golden):
    g = golden("cg")
    U = O.fermion_links(g["b_q"])
    x, it, _ = O.cg_normal(U, 0.05, g["b_b"], 1e-10, stop="batch_global")
    assert it == int(g["b_it_global"])
    assert rel_err(x, g["b_x_global"]) < 1e-12
    x, its, _ = O.cg_normal(U, 0.05, g["b_b"], 1e-10, stop="per_chain")
    assert np.array_equal(its, g["b_it_chain"])
    for c in range(4):
        assert rel_err(x[c], g["b_x_chain"][c]) < 1e-12


def test_oracle_cg_cap_raises(golden):
    g = golden("cg")
    U = O.fermion_links(g["a_q"])
    for stop in ("batch_global", "per_chain"):
        with pytest.raises(O.OracleSolverError) as err:
            O.cg_normal(U, 0.1, g["a_b"], 1e-10, maxiter=3, stop=stop)
        assert err.value.best_residual > 0


def test_oracle_cg_zero_rhs():
    U = O.fermion_links(np.zeros((2, 4, 4)))
    x, it, _ = O.cg_normal(U, 0.1, np.zeros((4, 4, 2), complex), 1e-12)
    assert it == 0 and np.all(x == 0)
    b = np.zeros((3, 4, 4, 2), complex)
    b[1] = 1.0
    U3 = O.fermion_links(np.zeros((3, 2, 4, 4)))
    x, its, _ = O.cg_normal(U3, 0.1, b, 1e-12, stop="per_chain")
    assert its[0] == 0 and its[2] == 0 and its[1] > 0
    assert np.all(x[0] == 0) and np.all(x[2] == 0)


@pytest.mark.parametrize("tag", ["u", "b"])
def test_oracle_forces_match_reference(golden, tag):
    g = golden("forces")
    q, eta, p = g[f"{tag}_q"], g[f"{tag}_eta"], g[f"{tag}_p"]
    beta, m0, tol = 2.0, 0.1, 1e-12
    U = O.fermion_links(q)
    chi, xi, _ = O.chi_xi(U, m0, eta, tol)
    assert rel_err(chi, g[f"{tag}_chi"]) < 1e-12
    assert rel_err(xi, g[f"{tag}_xi"]) < 1e-12
    f = O.fermion_force(U, chi, xi)
    assert rel_err(f, g[f"{tag}_f"]) < 1e-12
    b1, b2 = O.weighted_w_sums(U, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"])
    assert rel_err(b1, g[f"{tag}_b1"]) < 1e-14
    assert rel_err(b2, g[f"{tag}_b2"]) < 1e-14
    z1, z2 = O.z_pair(U, m0, g[f"{tag}_f"], g[f"{tag}_chi"], g[f"{tag}_xi"], tol)
    # measured 0.0: the oracle reproduces the reference's Z pair and FG terms exactly here
    assert rel_err(z1, g[f"{tag}_z1"]) < 1e-13
    assert rel_err(z2, g[f"{tag}_z2"]) < 1e-13
    fgff = O.fg_fermion_hessian_dot(U, m0, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_f"], tol)
    assert rel_err(fgff, g[f"{tag}_fgff"]) < 1e-13
    fggf = O.fg_fermion_hessian_dot(U, m0, g[f"{tag}_chi"], g[f"{tag}_xi"], g[f"{tag}_g"], tol)
    assert rel_err(fggf, g[f"{tag}_fggf"]) < 1e-13
    # real-arithmetic gauge pieces: bitwise
    assert np.array_equal(O.gauge_force(q, beta), g[f"{tag}_g"])
    assert np.array_equal(O.plaquette_angle(q), g[f"{tag}_plaq"])
    assert np.array_equal(O.fg_gauge_gauge(q, beta), g[f"{tag}_fggg"])
    assert np.array_equal(O.gauge_hessian_dot(q, beta, g[f"{tag}_f"]), g[f"{tag}_ghd"])
    assert np.array_equal(O.gauge_action(q, beta), g[f"{tag}_SG"])
    assert np.array_equal(O.avg_plaquette(q), g[f"{tag}_avgP"])
    assert np.array_equal(O.kinetic_energy(p), g[f"{tag}_kin"])
    assert np.array_equal(O.rotate_links(q, p, 0.37), g[f"{tag}_drift"])
    assert np.array_equal(O.wrap_angles(4.0 * q), g[f"{tag}_wrap"])
    sf = O.fermion_action(U, m0, eta, tol)
    assert rel_err(sf, g[f"{tag}_SF"]) < 1e-12


@pytest.mark.parametrize("tag", ["u", "b"])
def test_oracle_force_pieces_match_reference(golden, tag):
    """link_bilinears (both mu), oriented_plaquettes, plaquette_stencil."""
    g = golden("pieces")
    U = O.fermion_links(g[f"{tag}_q"])
    for mu in (0, 1):
        A, B = O.link_bilinears(U, mu, g[f"{tag}_a"], g[f"{tag}_b"])
        assert rel_err(A, g[f"{tag}_A{mu}"]) < 1e-14
        assert rel_err(B, g[f"{tag}_B{mu}"]) < 1e-14
    assert rel_err(O.oriented_plaquettes(g[f"{tag}_q"]), g[f"{tag}_P"]) < 1e-14
    assert rel_err(O.plaquette_stencil(g[f"{tag}_q"]), g[f"{tag}_stencil"]) < 1e-14


def test_oracle_measure_dh_matches_reference(golden):
    g = golden("measure")
    for k, scheme in enumerate(("adapted-nested-fg", "5stage-fg", "leapfrog")):
        cfg = O.Config(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                       micro_per_call=2 if scheme.startswith("adapted") else None,
                       cg_tol=1e-12, seed=11)
        rng = O.make_rng(11, k)
        q0 = 0.4 * rng.standard_normal((2, 6, 6))
        assert np.array_equal(q0, g[f"m{k}_q0"])
        m = O.measure_dh(q0, cfg, rng, n_samples=5)
        assert m["inversions_per_traj"] == int(g[f"m{k}_inv"])
        assert np.max(np.abs(m["dh"] - g[f"m{k}_dh"])) < 1e-10


def test_oracle_schemes_match_reference(golden):
    g = golden("traj")
    for k, scheme in enumerate(O.SCHEME_IDS):
        cfg = O.Config(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                       micro_per_call=2 if scheme in O.NESTED else None,
                       cg_tol=1e-12, seed=3)
        rng = O.make_rng(3, k)
        q = 0.4 * rng.standard_normal((2, 6, 6))
        assert np.array_equal(q, g[f"sch{k}_q0"])
        for t in range(2):
            q, s = O.hmc_update(q, cfg, rng)
            assert abs(s["dh"] - g[f"sch{k}_dh"][t]) < 1e-9, scheme
            assert s["accepted"] == bool(g[f"sch{k}_acc"][t])
            assert s["inversions"] == int(g[f"sch{k}_inv"][t])
        assert np.max(np.abs(q - g[f"sch{k}_qlast"])) < 1e-9


@pytest.mark.slow
@pytest.mark.parametrize("tag,h,n,bc", [("cfg1", 0.2, 20, "periodic"),
                                        ("cfg1h3", 1.0 / 3.0, 20, "periodic"),
                                        ("cfg1ap", 0.2, 5, "antiperiodic")])
def test_oracle_cfg1_trajectories(golden, tag, h, n, bc):
    """BASELINE configs[0]: dH to 1e-8 and the identical accept sequence."""
    g = golden("traj")
    cfg = O.Config(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=h, scheme="adapted-nested-fg",
                   micro_per_call=2, cg_tol=1e-10, seed=0, fermion_bc=bc)
    rng = O.make_rng(0, 0)
    q = O.hot_start(rng, 16, 16)
    assert np.array_equal(q, g[f"{tag}_q0"])
    for t in range(n):
        q, s = O.hmc_update(q, cfg, rng)
        assert abs(s["dh"] - g[f"{tag}_dh"][t]) < 1e-8
        assert s["accepted"] == bool(g[f"{tag}_acc"][t])
        assert s["inversions"] == int(g[f"{tag}_inv"][t])
    assert np.max(np.abs(q - g[f"{tag}_qlast"])) < 1e-8


def test_parallel_oracle_equals_serial_oracle():
    """oracle/parallel.py (the full-size checker) == the serial oracle: the
    per-chain CG of a chunked batch and independent hmc_update chains."""
    from oracle import parallel as OP
    rng = np.random.default_rng(7)
    B, L = 6, 8
    q = rng.uniform(-np.pi, np.pi, (B, 2, L, L))
    b = rng.standard_normal((B, L, L, 2)) + 1j * rng.standard_normal((B, L, L, 2))
    x, it = OP.cg_per_chain(q, b, 0.1, 1e-10, procs=2)
    for c in range(B):
        xs, its, _ = O.cg_normal(O.fermion_links(q[c]), 0.1, b[c], 1e-10)
        assert int(it[c]) == int(its[0] if np.ndim(its) else its)
        assert rel_err(x[c], xs) < 1e-13
    kw = dict(L=4, T=4, beta=2.0, m0=0.1, tau=0.5, h=0.25, scheme="adapted-nested-fg",
              micro_per_call=2, cg_tol=1e-10)
    ref = OP.hmc_chains([0, 3], 2024, kw, n_traj=2, procs=2)
    for c in (0, 3):
        r = O.make_rng(2024, c)
        qq = O.hot_start(r, 4, 4)
        assert np.array_equal(qq, ref[c][0])
        for t in range(2):
            qq, s = O.hmc_update(qq, O.Config(**kw), r)
            assert s["dh"] == ref[c][2][t] and s["accepted"] == ref[c][3][t]
        assert np.array_equal(qq, ref[c][1])


@pytest.mark.parametrize("scheme,h,micro", [("adapted-nested-fg", 0.25, 2), ("5stage", 0.2, None)])
def test_oracle_quenched_matches_reference(scheme, h, micro):
    """Quenched updates (eta = 0, no pseudofermion draw; hmc.py:79-80)
    against the reference's own run (tests/golden/make_quenched_golden.py)."""
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "quenched.npz")
    L = 12
    cfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=h, scheme=scheme, micro_per_call=micro,
                   cg_tol=1e-10, quenched=True)
    rng = O.make_rng(5, 0)
    q = O.hot_start(rng, L, L)
    assert np.array_equal(q, g[f"{scheme}_q0"])
    for k in range(3):
        q, st = O.hmc_update(q, cfg, rng)
        assert abs(st["dh"] - g[f"{scheme}_dh"][k]) < 1e-10
        assert st["accepted"] == bool(g[f"{scheme}_acc"][k])
        assert st["inversions"] == int(g[f"{scheme}_inv"][k])
    assert np.max(np.abs(q - g[f"{scheme}_q"])) < 1e-10
    m = O.measure_dh(g[f"{scheme}_q0"], cfg, O.make_rng(6, 1), 8)
    assert np.max(np.abs(m["dh"] - g[f"{scheme}_mdh"])) < 1e-10
    assert m["inversions_per_traj"] == int(g[f"{scheme}_minv"])


def test_oracle_thermalize_matches_reference():
    """thermalize (hmc.py:133-155) against the reference's own 60-update run
    with one step annealing (tests/golden/make_therm_golden.py)."""
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "therm.npz")
    cfg = O.Config(L=8, T=8, beta=1.0, m0=-0.231367, tau=1.0, h=0.1, cg_tol=1e-10,
                   n_thermalize=60, seed=11)
    q, hist = O.thermalize(cfg, O.make_rng(11, 0))
    assert np.max(np.abs(np.asarray(hist) - g["history"])) < 1e-10   # same NumPy arithmetic
    assert np.max(np.abs(q - g["q"])) < 1e-8
