"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
implementation itself (imported read-only from /root/reference/pkg/src).

This script runs only in the build container (the GPU box has no
/root/reference).  Its outputs are committed; the tests load them.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture records the inputs it was made from, so both the oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_*.py) can be
checked against the reference on identical inputs.
"""

from __future__ import annotations

import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
FIX = HERE.parent / "fixtures"
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF))

import schwinger as sw  # noqa: E402
from schwinger import fermion as F  # noqa: E402
from schwinger import gauge as G  # noqa: E402
from schwinger.integrators import MdState, integrate_trajectory, IntegratorSpec  # noqa: E402

M0_REF = -0.231367


def cspinor(rng, shape, scale=1.0):
    return scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))


class antiperiodic:
    """Context manager: the SURVEY §8(c) shim — flip the time links on the
    last time slice inside WilsonDirac only (fermions antiperiodic in t)."""

    def __enter__(self):
        self._orig = F.WilsonDirac.__init__

        def patched(obj, q, m0, _orig=self._orig):
            _orig(obj, q, m0)
            obj.U = obj.U.copy()
            obj.U[..., 1, :, -1] *= -1.0

        F.WilsonDirac.__init__ = patched
        return self

    def __exit__(self, *exc):
        F.WilsonDirac.__init__ = self._orig


def stencil_cases():
    out = {}
    cases = [
        # name, L, T, batch, m0, q generator
        ("s4", 4, 4, None, M0_REF, lambda r, s: 0.3 * r.standard_normal(s)),
        ("s16", 16, 16, None, 0.1, lambda r, s: r.uniform(-np.pi, np.pi, s)),
        ("b6x10", 6, 10, 3, 0.05, lambda r, s: r.uniform(-np.pi, np.pi, s)),
        ("s2", 2, 2, None, 0.3, lambda r, s: r.uniform(-np.pi, np.pi, s)),
        ("s3x5", 3, 5, 2, -0.1, lambda r, s: r.uniform(-np.pi, np.pi, s)),
        ("s32", 32, 32, 2, 0.1, lambda r, s: r.uniform(-np.pi, np.pi, s)),
    ]
    for i, (name, L, T, B, m0, gen) in enumerate(cases):
        rng = sw.make_rng(777, i)
        lshape = (2, L, T) if B is None else (B, 2, L, T)
        sshape = (L, T, 2) if B is None else (B, L, T, 2)
        q = gen(rng, lshape)
        psi = cspinor(rng, sshape)
        op = F.WilsonDirac(q, m0)
        out[f"{name}_q"] = q
        out[f"{name}_m0"] = np.float64(m0)
        out[f"{name}_psi"] = psi
        out[f"{name}_D"] = op.apply(psi)
        out[f"{name}_Ddag"] = op.apply_dag(psi)
        out[f"{name}_DdD"] = op.normal(psi)
    # antiperiodic-in-time shim on 8x8
    rng = sw.make_rng(777, 99)
    q = rng.uniform(-np.pi, np.pi, (2, 8, 8))
    psi = cspinor(rng, (8, 8, 2))
    with antiperiodic():
        op = F.WilsonDirac(q, 0.1)
        out["ap8_q"], out["ap8_m0"], out["ap8_psi"] = q, np.float64(0.1), psi
        out["ap8_D"], out["ap8_Ddag"], out["ap8_DdD"] = op.apply(psi), op.apply_dag(psi), op.normal(psi)
    np.savez_compressed(HERE / "stencil.npz", **out)


def cg_cases():
    out = {}
    # (a) cfg1-like single chain, 16x16 hot start, m0=0.1, tol=1e-10
    rng = sw.make_rng(0, 0)
    q = sw.hot_start(rng, sw.LatticeGeom(16, 16))
    b = cspinor(rng, (16, 16, 2))
    x, it, rel = F.cg_normal(F.WilsonDirac(q, 0.1), b, 1e-10)
    out.update(a_q=q, a_b=b, a_x=x, a_it=np.int64(it), a_rel=np.float64(rel))
    # (b) batch of 4 8x8 lattices: reference batched (global stop) and the
    #     same chains solved one at a time (per-chain semantics)
    rng = sw.make_rng(0, 1)
    q = rng.uniform(-np.pi, np.pi, (4, 2, 8, 8))
    b = cspinor(rng, (4, 8, 8, 2))
    b[2] *= 1e-3           # scale spread: per-chain targets differ
    x, it, rel = F.cg_normal(F.WilsonDirac(q, 0.05), b, 1e-10)
    out.update(b_q=q, b_b=b, b_x_global=x, b_it_global=np.int64(it), b_rel_global=np.float64(rel))
    xs, its = [], []
    for c in range(4):
        xc, itc, _ = F.cg_normal(F.WilsonDirac(q[c], 0.05), b[c], 1e-10)
        xs.append(xc)
        its.append(itc)
    out.update(b_x_chain=np.stack(xs), b_it_chain=np.array(its, dtype=np.int64))
    # (c) warm start x0 on 4x4, tol 1e-12, reference conftest-like field
    rng = sw.make_rng(0, 2)
    q = 0.3 * rng.standard_normal((2, 4, 4))
    b = cspinor(rng, (4, 4, 2))
    x0 = cspinor(rng, (4, 4, 2), 0.1)
    x, it, rel = F.cg_normal(F.WilsonDirac(q, M0_REF), b, 1e-12, x0=x0)
    out.update(c_q=q, c_b=b, c_x0=x0, c_x=x, c_it=np.int64(it))
    # (d) 32x32 hot start (one cfg2 batch element), m0=0.1, tol=1e-10
    rng = sw.make_rng(0, 3)
    q = sw.hot_start(rng, sw.LatticeGeom(32, 32))
    b = cspinor(rng, (32, 32, 2))
    x, it, rel = F.cg_normal(F.WilsonDirac(q, 0.1), b, 1e-10)
    out.update(d_q=q, d_b=b, d_x=x, d_it=np.int64(it), d_rel=np.float64(rel))
    # (e) a solve long enough to cross several residual replacements:
    #     light mass on a mild field, 12x12, tol 1e-12
    rng = sw.make_rng(0, 4)
    q = 0.2 * rng.standard_normal((2, 12, 12))
    b = cspinor(rng, (12, 12, 2))
    x, it, rel = F.cg_normal(F.WilsonDirac(q, M0_REF), b, 1e-12)
    out.update(e_q=q, e_b=b, e_x=x, e_it=np.int64(it))
    np.savez_compressed(HERE / "cg.npz", **out)
    print("cg iterations: a", out["a_it"], "b global", out["b_it_global"], "b chains",
          out["b_it_chain"], "c", out["c_it"], "d", out["d_it"], "e", out["e_it"])


def force_cases():
    out = {}
    for tag, B in (("u", None), ("b", 2)):
        rng = sw.make_rng(555, 0 if B is None else 1)
        L, T = 8, 8
        lshape = (2, L, T) if B is None else (B, 2, L, T)
        q = 0.7 * rng.standard_normal(lshape)
        eta = cspinor(rng, (L, T, 2) if B is None else (B, L, T, 2), 0.5)
        p = rng.standard_normal(lshape)
        beta, m0, tol = 2.0, 0.1, 1e-12
        op = F.WilsonDirac(q, m0)
        chi, xi, _ = F.chi_xi(op, eta, tol)
        f = F.fermion_force(op, chi, xi)
        g = G.gauge_force(q, beta)
        b1, b2 = F.weighted_w_sums(op, f, chi, xi)
        z1, z2 = F.z_pair(op, f, chi, xi, tol)
        fg_ff = F.fg_fermion_hessian_dot(op, chi, xi, f, tol)
        fg_gf = F.fg_fermion_hessian_dot(op, chi, xi, g, tol)
        out.update({f"{tag}_q": q, f"{tag}_eta": eta, f"{tag}_p": p,
                    f"{tag}_chi": chi, f"{tag}_xi": xi, f"{tag}_f": f, f"{tag}_g": g,
                    f"{tag}_b1": b1, f"{tag}_b2": b2, f"{tag}_z1": z1, f"{tag}_z2": z2,
                    f"{tag}_fgff": fg_ff, f"{tag}_fggf": fg_gf,
                    f"{tag}_fggg": G.fg_gauge_gauge(q, beta),
                    f"{tag}_ghd": G.gauge_hessian_dot(q, beta, f),
                    f"{tag}_plaq": G.plaq_angles(q),
                    f"{tag}_SG": np.asarray(G.gauge_action(q, beta)),
                    f"{tag}_avgP": np.asarray(G.avg_plaquette(q)),
                    f"{tag}_SF": np.asarray(F.fermion_action(op, eta, tol)),
                    f"{tag}_kin": np.asarray(sw.kinetic_energy(p)),
                    f"{tag}_drift": sw.rotate_links(q, p, 0.37),
                    f"{tag}_wrap": sw.wrap_angles(4.0 * q)})
    np.savez_compressed(HERE / "forces.npz", **out)


def piece_cases():
    """Building blocks of the force / force-gradient terms (fermion.py:317-327,
    gauge.py:62-95): link bilinears for both directions, the oriented
    plaquettes and the eight-plaquette stencil; unbatched and batched."""
    out = {}
    for tag, B in (("u", None), ("b", 3)):
        rng = sw.make_rng(777, 0 if B is None else 1)
        L, T = 6, 10
        lshape = (2, L, T) if B is None else (B, 2, L, T)
        sshape = (L, T, 2) if B is None else (B, L, T, 2)
        q = rng.uniform(-np.pi, np.pi, lshape)
        a, b = cspinor(rng, sshape), cspinor(rng, sshape)
        op = F.WilsonDirac(q, 0.1)
        for mu in (0, 1):
            A, Bb = F.link_bilinears(op, mu, a, b)
            out[f"{tag}_A{mu}"], out[f"{tag}_B{mu}"] = A, Bb
        out.update({f"{tag}_q": q, f"{tag}_a": a, f"{tag}_b": b,
                    f"{tag}_P": G.oriented_plaquettes(q), f"{tag}_stencil": G.plaquette_stencil(q)})
    np.savez_compressed(HERE / "pieces.npz", **out)


def run_chain(q, cfg, rng, n):
    dh, acc, inv, qs = [], [], [], []
    for _ in range(n):
        q, st = sw.hmc_update(q, cfg, rng)
        dh.append(st.dh)
        acc.append(st.accepted)
        inv.append(st.inversions)
        qs.append(q)
    return np.array(dh), np.array(acc), np.array(inv), np.stack(qs)


def traj_cases():
    out = {}
    base = sw.HmcConfig(L=16, T=16, beta=2.0, m0=0.1, tau=1.0, h=0.2,
                        scheme="adapted-nested-fg", micro_per_call=2, cg_tol=1e-10,
                        seed=0, n_thermalize=0, n_samples=1)
    for tag, cfg, n, ap in (("cfg1", base, 20, False),
                            ("cfg1h3", replace(base, h=1.0 / 3.0), 20, False),
                            ("cfg1ap", base, 5, True)):
        t0 = time.time()
        rng = sw.make_rng(0, 0)
        q0 = sw.hot_start(rng, sw.LatticeGeom(16, 16))
        if ap:
            with antiperiodic():
                dh, acc, inv, qs = run_chain(q0, cfg, rng, n)
        else:
            dh, acc, inv, qs = run_chain(q0, cfg, rng, n)
        out.update({f"{tag}_q0": q0, f"{tag}_dh": dh, f"{tag}_acc": acc,
                    f"{tag}_inv": inv, f"{tag}_qfirst": qs[0], f"{tag}_qlast": qs[-1]})
        print(f"{tag}: {n} traj in {time.time() - t0:.1f}s, acc {acc.sum()}/{n}, "
              f"dh {np.round(dh, 5).tolist()}")
    # every scheme, 2 trajectories each on a mild 6x6 field
    for k, scheme in enumerate(sw.SCHEME_IDS):
        cfg = sw.HmcConfig(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                           micro_per_call=2 if scheme in
                           ("nested-leapfrog", "nested-5stage", "nested-fg", "adapted-nested-fg") else None,
                           cg_tol=1e-12, seed=3)
        rng = sw.make_rng(3, k)
        q0 = 0.4 * rng.standard_normal((2, 6, 6))
        dh, acc, inv, qs = run_chain(q0, cfg, rng, 2)
        out.update({f"sch{k}_q0": q0, f"sch{k}_dh": dh, f"sch{k}_acc": acc,
                    f"sch{k}_inv": inv, f"sch{k}_qlast": qs[-1]})
    out["schemes"] = np.array(sw.SCHEME_IDS)
    np.savez_compressed(HERE / "traj.npz", **out)


def measure_cases():
    out = {}
    for k, scheme in enumerate(("adapted-nested-fg", "5stage-fg", "leapfrog")):
        cfg = sw.HmcConfig(L=6, T=6, beta=1.0, m0=0.1, tau=0.5, h=0.25, scheme=scheme,
                           micro_per_call=2 if scheme.startswith("adapted") else None,
                           cg_tol=1e-12, seed=11)
        rng = sw.make_rng(11, k)
        q0 = 0.4 * rng.standard_normal((2, 6, 6))
        m = sw.measure_dh(q0, cfg, rng, n_samples=5)
        out.update({f"m{k}_q0": q0, f"m{k}_dh": m.dh, f"m{k}_inv": np.int64(m.inversions_per_traj),
                    f"m{k}_acc": np.float64(m.acceptance)})
    np.savez_compressed(HERE / "measure.npz", **out)


def therm_fixture():
    path = FIX / "therm_8x8.cfg"
    if path.exists():
        return
    FIX.mkdir(parents=True, exist_ok=True)
    cfg = sw.desk_scale(sw.HmcConfig())
    t0 = time.time()
    q, hist = sw.thermalize(cfg, sw.make_rng(cfg.seed, 0))
    sw.save_gauge_config(path, q, cfg.beta, cfg.m0, cfg.seed)
    print(f"therm_8x8: {time.time() - t0:.1f}s, final plaquette {hist[-1]:.5f}")


if __name__ == "__main__":
    which = sys.argv[1:] or ["stencil", "cg", "force", "pieces", "traj", "measure", "therm"]
    for w in which:
        dict(stencil=stencil_cases, cg=cg_cases, force=force_cases, pieces=piece_cases,
             traj=traj_cases, measure=measure_cases, therm=therm_fixture)[w]()
