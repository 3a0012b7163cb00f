"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 path. Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` legs
of ``bench.py`` may import it; the product package never does.

It is an independent NumPy restatement of the reference HMC molecular-dynamics
path of arXiv:1512.03812's Schwinger-model package (``/root/reference/pkg/src/
schwinger``), written as site-plane formulas (Appendix A of SURVEY.md) rather
than a transcription.  Every function cites the reference ``file:line`` whose
behaviour it restates.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (imported
from /root/reference in the build container) on seeded inputs and commits the
outputs as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this
oracle against them (bit-level where the reference is real arithmetic, 1e-13
relative for complex stencils, identical CG iteration counts and accept
sequences for trajectories).

Layouts (identical to the reference, lattice.py:3-12):
  link fields   float64  (..., 2, L, T)   direction first, x then t
  spinor fields complex128 (..., L, T, 2)
  direction 0 = x (axis -2 of a site plane), 1 = t (axis -1)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

TWO_PI = 2.0 * np.pi
DEFAULT_TOL = 1e-12          # fermion.py:28
DEFAULT_MAXITER = 10_000     # fermion.py:29
RESIDUAL_REPLACEMENT = 50    # fermion.py:199
FG_KICK_SIGN = -1.0          # integrators.py:30
DEFAULT_FG_COEFF = 1.0 / 72.0  # integrators.py:32

# 11-stage coefficients (integrators.py:40-43)
ELEVEN = dict(sigma=0.08398315262876693, eta=0.2539785108410595,
              lam=0.6822365335719091, theta=-0.03230286765269967)

SCHEME_IDS = ("leapfrog", "5stage", "5stage-fg", "fg-approx", "11stage",
              "nested-leapfrog", "nested-5stage", "nested-fg",
              "adapted-nested-fg")                       # integrators.py:61-63
NESTED = ("nested-leapfrog", "nested-5stage", "nested-fg", "adapted-nested-fg")
INVERSIONS_PER_STEP = {"leapfrog": 4, "5stage": 6, "5stage-fg": 10,
                       "fg-approx": 8, "11stage": 12, "nested-leapfrog": 4,
                       "nested-5stage": 6, "nested-fg": 8,
                       "adapted-nested-fg": 8}           # integrators.py:69-79


class OracleSolverError(RuntimeError):
    """CG iteration cap (fermion.py:63-68)."""

    def __init__(self, message, best_residual):
        super().__init__(f"{message} (best relative residual {best_residual:.3e})")
        self.best_residual = best_residual


# ---------------------------------------------------------------------------
# site-plane neighbour access.  A "plane" is (..., L, T); mu selects the axis.
# ---------------------------------------------------------------------------

def _ax(mu):
    return -2 if mu == 0 else -1


def at_fwd(a, mu, k=1):
    """a(n + k*mu) on a periodic plane."""
    return np.roll(a, -k, axis=_ax(mu))


def at_bwd(a, mu, k=1):
    """a(n - k*mu) on a periodic plane."""
    return np.roll(a, k, axis=_ax(mu))


# ---------------------------------------------------------------------------
# L0: angles, RNG, momenta (lattice.py)
# ---------------------------------------------------------------------------

def wrap_angles(q):
    """Floored reduction to [-pi, pi) (lattice.py:28-30)."""
    return np.mod(q + np.pi, TWO_PI) - np.pi


def rotate_links(q, p, h):
    """q -> wrap(q + h p) (lattice.py:111-118)."""
    return wrap_angles(q + h * p)


def kinetic_energy(p):
    """(1/2) sum p^2 per sample (lattice.py:128-130)."""
    return 0.5 * np.sum(p * p, axis=(-3, -2, -1))


def make_rng(seed, stream=0):
    """Philox(key=[seed, stream]) generator (lattice.py:86-89)."""
    key = np.array([seed % 2**64, stream % 2**64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def hot_start(rng, L, T, batch=None):
    """theta ~ U(-pi, pi) per link (lattice.py:102-104)."""
    shape = (2, L, T) if batch is None else (batch, 2, L, T)
    return rng.uniform(-np.pi, np.pi, size=shape)


def sample_momenta(rng, L, T, batch=None):
    """N(0,1) per link (lattice.py:92-95)."""
    shape = (2, L, T) if batch is None else (batch, 2, L, T)
    return rng.standard_normal(shape)


def load_gauge_config(path):
    """Reader for the 'schwinger-u1 v1' file format (lattice.py:157-172)."""
    with open(path, "rb") as fh:
        head = fh.readline().decode("ascii").split()
        body = fh.read()
    L, T = int(head[2]), int(head[3])
    arr = np.frombuffer(body, dtype="<f8").reshape(T, L, 2)
    meta = dict(L=L, T=T, beta=float(head[4]), m0=float(head[5]), seed=int(head[6]))
    return np.ascontiguousarray(arr.transpose(2, 1, 0)), meta


# ---------------------------------------------------------------------------
# L1a: gauge sector (gauge.py)
# ---------------------------------------------------------------------------

def plaquette_angle(q):
    """theta(n) = q0(n) + q1(n+x) - q0(n+t) - q1(n)  (gauge.py:21-24)."""
    q0, q1 = q[..., 0, :, :], q[..., 1, :, :]
    return q0 + at_fwd(q1, 0) - at_fwd(q0, 1) - q1


def gauge_action(q, beta):
    """beta * sum(1 - cos theta)  (gauge.py:37-40)."""
    return beta * np.sum(1.0 - np.cos(plaquette_angle(q)), axis=(-2, -1))


def avg_plaquette(q):
    """mean cos theta (gauge.py:32-34)."""
    return np.mean(np.cos(plaquette_angle(q)), axis=(-2, -1))


def gauge_force(q, beta):
    """beta * g with g0 = s - s(n-t), g1 = s(n-x) - s  (gauge.py:43-59)."""
    s = np.sin(plaquette_angle(q))
    g = np.empty_like(q)
    g[..., 0, :, :] = s - at_bwd(s, 1)
    g[..., 1, :, :] = at_bwd(s, 0) - s
    return beta * g


def _oriented_plaquette(q, mu):
    """P1 for links of direction mu: e^{i theta}, conjugated for mu=1
    (gauge.py:62-67)."""
    z = np.exp(1j * plaquette_angle(q))
    return z if mu == 0 else np.conj(z)


def oriented_plaquettes(q):
    """P1(n, mu) stacked over mu, shape (..., 2, L, T) (gauge.py:62-67)."""
    return np.stack([_oriented_plaquette(q, 0), _oriented_plaquette(q, 1)], axis=-3)


def plaquette_stencil(q):
    """The eight translates P1..P8 of the mu-oriented plaquette attached to
    link (n, mu), shape (8, ..., 2, L, T) (gauge.py:70-95):
    P2 = P1(n-nu), P3 = P1(n+mu), P4 = P1(n+nu), P5 = P1(n-mu),
    P6 = P1(n-mu-nu), P7 = P1(n-2nu), P8 = P1(n+mu-nu)."""
    p1 = oriented_plaquettes(q)
    out = np.empty((8,) + p1.shape, dtype=p1.dtype)
    for mu in (0, 1):
        nu = 1 - mu
        base = p1[..., mu, :, :]
        out[0, ..., mu, :, :] = base
        out[1, ..., mu, :, :] = at_bwd(base, nu)
        out[2, ..., mu, :, :] = at_fwd(base, mu)
        out[3, ..., mu, :, :] = at_fwd(base, nu)
        out[4, ..., mu, :, :] = at_bwd(base, mu)
        out[5, ..., mu, :, :] = at_bwd(at_bwd(base, mu), nu)
        out[6, ..., mu, :, :] = at_bwd(base, nu, 2)
        out[7, ..., mu, :, :] = at_bwd(at_fwd(base, mu), nu)
    return out


def fg_gauge_gauge(q, beta):
    """Closed-form C_GG from the eight translated plaquettes
    (gauge.py:70-107)."""
    out = np.empty_like(q)
    for mu in (0, 1):
        nu = 1 - mu
        p1 = _oriented_plaquette(q, mu)
        p2 = at_bwd(p1, nu)                       # P1(n - nu)
        p3 = at_fwd(p1, mu)                       # P1(n + mu)
        p4 = at_fwd(p1, nu)                       # P1(n + nu)
        p5 = at_bwd(p1, mu)                       # P1(n - mu)
        p6 = at_bwd(at_bwd(p1, mu), nu)           # P1(n - mu - nu)
        p7 = at_bwd(p1, nu, 2)                    # P1(n - 2 nu)
        p8 = at_bwd(at_fwd(p1, mu), nu)           # P1(n + mu - nu)
        first = np.imag(4.0 * p1 - p2 - p3 - p4 - p5) * np.real(p1)
        second = np.imag(4.0 * p2 - p1 - p6 - p7 - p8) * np.real(p2)
        out[..., mu, :, :] = first - second
    return 2.0 * beta * beta * out


def gauge_hessian_dot(q, beta, w):
    """2 * sum w * Hess(S_G), closed form (gauge.py:110-136)."""
    if q.shape[-3:] != w.shape[-3:]:
        raise ValueError("link/weight shape mismatch")
    c = np.cos(plaquette_angle(q))
    out = np.empty(np.broadcast_shapes(q.shape, w.shape))
    for mu in (0, 1):
        nu = 1 - mu
        wm, wn = w[..., mu, :, :], w[..., nu, :, :]
        a = wm + at_fwd(wn, mu) - at_fwd(wm, nu) - wn
        b = wm - at_bwd(at_fwd(wn, mu), nu) - at_bwd(wm, nu) + at_bwd(wn, nu)
        out[..., mu, :, :] = 2.0 * beta * (a * c + b * at_bwd(c, nu))
    return out


# ---------------------------------------------------------------------------
# L1b: Wilson fermions (fermion.py)
# ---------------------------------------------------------------------------

# Rank-1 projector table (fermion.py:36-51):  (1 + sgn*sigma_mu) v = (w, e*w)
# with w = v0 + c*v1.  Key: (mu, sgn).
_PROJ = {(0, -1): (-1.0, -1.0), (1, -1): (1j, -1j),
         (0, +1): (1.0, 1.0), (1, +1): (-1j, 1j)}


def _w(v0, v1, mu, sgn):
    c, _ = _PROJ[(mu, sgn)]
    if c == -1.0:
        return v0 - v1
    if c == 1.0:
        return v0 + v1
    return v0 + c * v1


def fermion_links(q, bc="periodic"):
    """U = exp(i q) (fermion.py:94).  ``bc='antiperiodic'`` flips the sign of
    the time links on the last time slice (BASELINE.json configs[0]); not a
    reference feature, see DESIGN.md."""
    u = np.exp(1j * q)
    if bc == "antiperiodic":
        u = u.copy()
        u[..., 1, :, -1] *= -1.0
    elif bc != "periodic":
        raise ValueError(f"unknown fermion bc {bc!r}")
    return u


def dirac(U, psi, m0, dagger=False):
    """(D psi) or (D^dag psi) per Appendix A2 (fermion.py:101-127)."""
    v0, v1 = psi[..., 0], psi[..., 1]
    fwd_sgn, bwd_sgn = (+1, -1) if dagger else (-1, +1)
    s0 = s1 = 0.0
    for mu in (0, 1):
        u = U[..., mu, :, :]
        e_f = _PROJ[(mu, fwd_sgn)][1]
        e_b = _PROJ[(mu, bwd_sgn)][1]
        hop_f = u * at_fwd(_w(v0, v1, mu, fwd_sgn), mu)
        hop_b = at_bwd(np.conj(u) * _w(v0, v1, mu, bwd_sgn), mu)
        s0 = s0 + hop_f + hop_b
        s1 = s1 + e_f * hop_f + e_b * hop_b
    d = 2.0 + m0
    return np.stack([d * v0 - 0.5 * s0, d * v1 - 0.5 * s1], axis=-1)


def normal_op(U, psi, m0):
    """D^dag D psi (fermion.py:129-131)."""
    return dirac(U, dirac(U, psi, m0), m0, dagger=True)


def sdot(a, b):
    """sum conj(a) b over sites and spin (fermion.py:54-56)."""
    return np.sum(np.conj(a) * b, axis=(-3, -2, -1))


def _chain(v):
    return np.asarray(v)[..., None, None, None]


def cg_normal(U, m0, b, tol, maxiter=DEFAULT_MAXITER, x0=None,
              stop="batch_global"):
    """CG on D^dag D x = b (fermion.py:171-217).

    stop='batch_global' is the reference's batched semantics (every chain
    iterates until all pass; the true-residual re-check and the residual
    reset act on the whole batch).  stop='per_chain' is the semantics of
    calling the reference once per chain (hmc_update), expressed with masks.

    Returns (x, iterations, worst relative residual); iterations is an int for
    batch_global and an int array (per chain) for per_chain.
    """
    A = lambda v: normal_op(U, v, m0)
    normb = np.sqrt(np.real(sdot(b, b)))
    target = tol * normb
    if stop == "batch_global":
        if np.all(normb == 0.0):
            return np.zeros_like(b), 0, 0.0
    elif stop != "per_chain":
        raise ValueError(stop)

    x = np.zeros_like(b) if x0 is None else x0.astype(np.complex128, copy=True)
    r = b.copy() if x0 is None else b - A(x)
    p = r.copy()
    rs = np.real(sdot(r, r))
    safe_nb = np.where(normb > 0, normb, 1.0)

    if stop == "batch_global":
        best = np.inf
        for it in range(1, maxiter + 1):
            ap = A(p)
            den = np.real(sdot(p, ap))
            alpha = np.where(den > 0.0, rs / np.where(den > 0.0, den, 1.0), 0.0)
            x = x + _chain(alpha) * p
            r = b - A(x) if it % RESIDUAL_REPLACEMENT == 0 else r - _chain(alpha) * ap
            rs_new = np.real(sdot(r, r))
            if np.all(np.sqrt(rs_new) <= target):
                tr = b - A(x)
                tn = np.sqrt(np.real(sdot(tr, tr)))
                best = float(np.max(np.where(normb > 0, tn / safe_nb, 0.0)))
                if np.all(tn <= target):
                    return x, it, best
                r = tr
                rs_new = np.real(sdot(r, r))
            beta = np.where(rs > 0.0, rs_new / np.where(rs > 0.0, rs, 1.0), 0.0)
            p = r + _chain(beta) * p
            rs = rs_new
        rel = np.max(np.sqrt(rs) / safe_nb)
        raise OracleSolverError(f"CG exceeded {maxiter} iterations", min(best, float(rel)))

    # per-chain: each chain is an independent unbatched solve
    scalar = b.ndim == 3
    done = np.atleast_1d(normb == 0.0).copy()
    iters = np.zeros(done.shape, dtype=np.int64)
    relres = np.zeros(done.shape)
    if scalar:
        x, r, p = x[None], r[None], p[None]
        b_ = b[None]
        rs, target, normb_, safe_ = (np.atleast_1d(v) for v in (rs, target, normb, safe_nb))
    else:
        b_, normb_, safe_ = b, normb, safe_nb
    if np.any(done):
        x[done] = 0.0
    for it in range(1, maxiter + 1):
        if np.all(done):
            break
        live = ~done
        ap = A(p)
        den = np.real(sdot(p, ap))
        alpha = np.where(den > 0.0, rs / np.where(den > 0.0, den, 1.0), 0.0)
        alpha = np.where(live, alpha, 0.0)
        x_new = x + _chain(alpha) * p
        x = np.where(_chain(live), x_new, x)
        if it % RESIDUAL_REPLACEMENT == 0:
            r_new = b_ - A(x)
        else:
            r_new = r - _chain(alpha) * ap
        r = np.where(_chain(live), r_new, r)
        rs_new = np.real(sdot(r, r))
        check = live & (np.sqrt(rs_new) <= target)
        if np.any(check):
            tr = b_ - A(x)
            tn = np.sqrt(np.real(sdot(tr, tr)))
            conv = check & (tn <= target)
            iters[conv] = it
            relres[conv] = np.where(normb_ > 0, tn / safe_, 0.0)[conv]
            retry = check & ~conv
            r = np.where(_chain(retry), tr, r)
            rs_new = np.where(retry, np.real(sdot(tr, tr)), rs_new)
            done = done | conv
        beta = np.where(rs > 0.0, rs_new / np.where(rs > 0.0, rs, 1.0), 0.0)
        p = np.where(_chain(live), r + _chain(beta) * p, p)
        rs = np.where(live, rs_new, rs)
    if not np.all(done):
        rel = float(np.max(np.sqrt(rs) / safe_))
        raise OracleSolverError(f"CG exceeded {maxiter} iterations", rel)
    if scalar:
        return x[0], iters, float(relres.max())
    return x, iters, float(relres.max())


class Counter:
    """Inversion tally (fermion.py:71-78)."""

    def __init__(self):
        self.count = 0

    def add(self, n):
        self.count += n


def solve_normal(U, m0, b, tol, counter=None, stop="batch_global", x0=None,
                 maxiter=DEFAULT_MAXITER):
    """(D^dag D)^{-1} b; two inversions (fermion.py:233-242)."""
    x, it, _ = cg_normal(U, m0, b, tol, maxiter=maxiter, x0=x0, stop=stop)
    if counter is not None:
        counter.add(2)
    return x, it


def solve_dirac(U, m0, b, tol, counter=None, stop="batch_global"):
    """D^{-1} b = CG(D^dag D, D^dag b); one inversion (fermion.py:245-259)."""
    x, it, _ = cg_normal(U, m0, dirac(U, b, m0, dagger=True), tol, stop=stop)
    if counter is not None:
        counter.add(1)
    return x, it


def solve_dirac_dagger(U, m0, b, tol, counter=None, stop="batch_global"):
    """D^{-dag} b = D CG(D^dag D, b); one inversion (fermion.py:262-276)."""
    y, it, _ = cg_normal(U, m0, b, tol, stop=stop)
    if counter is not None:
        counter.add(1)
    return dirac(U, y, m0), it


def chi_xi(U, m0, eta, tol, counter=None, stop="batch_global"):
    """xi = (D^dag D)^{-1} eta, chi = D xi (fermion.py:300-310)."""
    xi, it = solve_normal(U, m0, eta, tol, counter, stop)
    return dirac(U, xi, m0), xi, it


def fermion_action(U, m0, eta, tol, counter=None, stop="batch_global"):
    """Re <eta, (D^dag D)^{-1} eta> (fermion.py:293-297)."""
    x, _ = solve_normal(U, m0, eta, tol, counter, stop)
    return np.real(sdot(eta, x))


def _bilinears(U, mu, a, b):
    """A(n) = conj(w-(a)(n)) U w-(b)(n+mu);
    B(n) = conj(w+(a)(n+mu)) conj(U) w+(b)(n)   (fermion.py:317-327)."""
    u = U[..., mu, :, :]
    a0, a1, b0, b1 = a[..., 0], a[..., 1], b[..., 0], b[..., 1]
    A_ = np.conj(_w(a0, a1, mu, -1)) * u * at_fwd(_w(b0, b1, mu, -1), mu)
    B_ = np.conj(at_fwd(_w(a0, a1, mu, +1), mu)) * np.conj(u) * _w(b0, b1, mu, +1)
    return A_, B_


def link_bilinears(U, mu, a, b):
    """(A, B) hopping contractions attached to link (n, mu) (fermion.py:317-327)."""
    return _bilinears(U, mu, a, b)


def fermion_force(U, chi, xi):
    """f(n,mu) = -Im[A - B] (fermion.py:330-336)."""
    parts = []
    for mu in (0, 1):
        A_, B_ = _bilinears(U, mu, chi, xi)
        parts.append(-np.imag(A_ - B_))
    return np.stack(parts, axis=-3)


def weighted_w_sums(U, weight, chi, xi):
    """b1 = sum weight*w1, b2 = sum weight*w2 as spinor fields
    (fermion.py:362-383)."""
    shp = np.broadcast_shapes(chi.shape, xi.shape)
    b1 = np.zeros(shp, dtype=np.complex128)
    b2 = np.zeros(shp, dtype=np.complex128)
    c0, c1, x0_, x1_ = chi[..., 0], chi[..., 1], xi[..., 0], xi[..., 1]
    for nu in (0, 1):
        u = U[..., nu, :, :]
        wt = weight[..., nu, :, :]
        e_m, e_p = _PROJ[(nu, -1)][1], _PROJ[(nu, +1)][1]
        t1 = 0.5j * at_bwd(wt * np.conj(u) * _w(c0, c1, nu, -1), nu)
        t2 = -0.5j * wt * u * at_fwd(_w(c0, c1, nu, +1), nu)
        b1[..., 0] += t1 + t2
        b1[..., 1] += e_m * t1 + e_p * t2
        t3 = -0.5j * wt * u * at_fwd(_w(x0_, x1_, nu, -1), nu)
        t4 = 0.5j * at_bwd(wt * np.conj(u) * _w(x0_, x1_, nu, +1), nu)
        b2[..., 0] += t3 + t4
        b2[..., 1] += e_m * t3 + e_p * t4
    return b1, b2


def z_pair(U, m0, weight, chi, xi, tol, counter=None, stop="batch_global"):
    """Z1 = D^{-dag} b1, Z2 = D^{-1}(b2 + Z1) (fermion.py:386-394)."""
    b1, b2 = weighted_w_sums(U, weight, chi, xi)
    z1, _ = solve_dirac_dagger(U, m0, b1, tol, counter, stop)
    z2, _ = solve_dirac(U, m0, b2 + z1, tol, counter, stop)
    return z1, z2


def fg_fermion_hessian_dot(U, m0, chi, xi, weight, tol, counter=None,
                           stop="batch_global"):
    """C = 2Im(A[Z1,xi]-B[Z1,xi]) + 2Im(A[chi,Z2]-B[chi,Z2])
           - 2Re(A[chi,xi]+B[chi,xi]) * weight   (fermion.py:397-417)."""
    z1, z2 = z_pair(U, m0, weight, chi, xi, tol, counter, stop)
    parts = []
    for mu in (0, 1):
        a1, b1 = _bilinears(U, mu, z1, xi)
        a2, b2 = _bilinears(U, mu, chi, z2)
        a3, b3 = _bilinears(U, mu, chi, xi)
        parts.append(2.0 * np.imag(a1 - b1) + 2.0 * np.imag(a2 - b2)
                     - 2.0 * np.real(a3 + b3) * weight[..., mu, :, :])
    return np.stack(parts, axis=-3)


def pseudofermion_heatbath(U, m0, rng, L, T, batch=None):
    """eta = D^dag phi, phi = (N + iN)/sqrt 2, real part drawn first
    (fermion.py:283-290)."""
    shape = (L, T, 2) if batch is None else (batch, L, T, 2)
    re = rng.standard_normal(shape)
    im = rng.standard_normal(shape)
    phi = (re + 1j * im) / np.sqrt(2.0)
    return dirac(U, phi, m0, dagger=True)


# ---------------------------------------------------------------------------
# L2: integrators (integrators.py) as schedule tables
# ---------------------------------------------------------------------------

@dataclass
class State:
    """MD state (integrators.py:82-104)."""
    q: np.ndarray
    p: np.ndarray
    eta: np.ndarray
    beta: float
    m0: float
    tol: float = DEFAULT_TOL
    counter: Counter = field(default_factory=Counter)
    bc: str = "periodic"
    stop: str = "batch_global"


def _links(st, q=None):
    return fermion_links(st.q if q is None else q, st.bc)


def _solve_pair(st, q=None):
    U = _links(st, q)
    chi, xi, _ = chi_xi(U, st.m0, st.eta, st.tol, st.counter, st.stop)
    return U, chi, xi


def op_drift(st, dt):                                   # integrators.py:157-158
    st.q = rotate_links(st.q, st.p, dt)


def op_kick(st, kind, dt):                              # integrators.py:161-186
    if dt == 0.0:
        return
    if kind == "gauge":
        st.p = st.p - dt * gauge_force(st.q, st.beta)
        return
    U, chi, xi = _solve_pair(st)
    f = fermion_force(U, chi, xi)
    if kind == "full":
        f = gauge_force(st.q, st.beta) + f
    st.p = st.p - dt * f


def op_fg_kick(st, kind, b_dt, c_dt3):                 # integrators.py:189-246
    if c_dt3 == 0.0:
        op_kick(st, {"gauge": "gauge", "fermion": "fermion"}.get(kind, "full"), b_dt)
        return
    sc = FG_KICK_SIGN * c_dt3
    if kind == "gauge":
        st.p = st.p - (b_dt * gauge_force(st.q, st.beta) + sc * fg_gauge_gauge(st.q, st.beta))
        return
    U, chi, xi = _solve_pair(st)
    f = fermion_force(U, chi, xi)
    if kind == "fermion":
        fg = fg_fermion_hessian_dot(U, st.m0, chi, xi, f, st.tol, st.counter, st.stop)
        st.p = st.p - (b_dt * f + sc * fg)
    elif kind == "full":
        g = gauge_force(st.q, st.beta)
        fg = (fg_gauge_gauge(st.q, st.beta) + gauge_hessian_dot(st.q, st.beta, f)
              + fg_fermion_hessian_dot(U, st.m0, chi, xi, g, st.tol, st.counter, st.stop)
              + fg_fermion_hessian_dot(U, st.m0, chi, xi, f, st.tol, st.counter, st.stop))
        st.p = st.p - (b_dt * (g + f) + sc * fg)
    elif kind == "approx":
        force = gauge_force(st.q, st.beta) + f
        qs = rotate_links(st.q, force, 2.0 * FG_KICK_SIGN * c_dt3 / b_dt)
        U2, chi2, xi2 = _solve_pair(st, qs)
        shifted = gauge_force(qs, st.beta) + fermion_force(U2, chi2, xi2)
        st.p = st.p - b_dt * shifted
    else:
        raise ValueError(kind)


def op_inner(st, kind, span, m, fgc):                   # integrators.py:253-271
    d = span / m
    for _ in range(m):
        if kind == "leapfrog":
            op_kick(st, "gauge", 0.5 * d)
            op_drift(st, d)
            op_kick(st, "gauge", 0.5 * d)
        else:
            op_kick(st, "gauge", d / 6.0)
            op_drift(st, 0.5 * d)
            op_fg_kick(st, "gauge", 2.0 * d / 3.0, fgc * d**3)
            op_drift(st, 0.5 * d)
            op_kick(st, "gauge", d / 6.0)


def macro_step(st, scheme, h, m, fgc):
    """One macro step of ``scheme`` (integrators.py:278-349)."""
    c3 = fgc * h**3
    if scheme == "leapfrog":
        op_kick(st, "full", 0.5 * h); op_drift(st, h); op_kick(st, "full", 0.5 * h)
    elif scheme in ("5stage", "5stage-fg", "fg-approx"):
        op_kick(st, "full", h / 6.0)
        op_drift(st, 0.5 * h)
        if scheme == "5stage":
            op_kick(st, "full", 2.0 * h / 3.0)
        else:
            op_fg_kick(st, "full" if scheme == "5stage-fg" else "approx", 2.0 * h / 3.0, c3)
        op_drift(st, 0.5 * h)
        op_kick(st, "full", h / 6.0)
    elif scheme == "11stage":
        s, e, l, t = (ELEVEN[k] for k in ("sigma", "eta", "lam", "theta"))
        w_half = 0.5 * (1.0 - 2.0 * (l + s))
        c_mid = 1.0 - 2.0 * (t + e)
        seq = ((s, e), (l, t), (w_half, c_mid), (w_half, t), (l, e), (s, None))
        for kw, dw in seq:
            op_kick(st, "full", kw * h)
            if dw is not None:
                op_drift(st, dw * h)
    elif scheme == "nested-leapfrog":
        op_kick(st, "fermion", 0.5 * h); op_inner(st, "leapfrog", h, m, fgc)
        op_kick(st, "fermion", 0.5 * h)
    else:
        inner = "fg" if scheme == "nested-fg" else "leapfrog"
        op_kick(st, "fermion", h / 6.0)
        op_inner(st, inner, 0.5 * h, m, fgc)
        if scheme == "nested-5stage":
            op_kick(st, "fermion", 2.0 * h / 3.0)
        else:
            op_fg_kick(st, "fermion", 2.0 * h / 3.0, c3)
        op_inner(st, inner, 0.5 * h, m, fgc)
        op_kick(st, "fermion", h / 6.0)


def micro_steps(scheme, micro_per_call=None, micro_ratio=10.0):
    """integrators.py:135-143."""
    if scheme not in NESTED:
        return 1
    if micro_per_call is not None:
        return micro_per_call
    span = 1.0 if scheme == "nested-leapfrog" else 0.5
    return max(1, round(span * micro_ratio))


def integrate(st, scheme, h, tau, micro_per_call=None, micro_ratio=10.0,
              fgc=DEFAULT_FG_COEFF):
    """integrate_trajectory (integrators.py:365-382): returns (n_steps, inversions)."""
    if not tau > 0:
        raise ValueError("tau must be positive")
    n = max(1, round(tau / h))
    m = micro_steps(scheme, micro_per_call, micro_ratio)
    before = st.counter.count
    for _ in range(n):
        macro_step(st, scheme, h, m, fgc)
    return n, st.counter.count - before


# ---------------------------------------------------------------------------
# L3: HMC driver (hmc.py)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    """Mirror of HmcConfig (config.py:18-43) with the extra fermion_bc flag."""
    L: int = 32
    T: int = 32
    beta: float = 1.0
    m0: float = -0.231367
    tau: float = 2.0
    h: float = 0.05
    scheme: str = "leapfrog"
    micro_per_call: int | None = None
    micro_ratio: float = 10.0
    cg_tol: float = 1e-12
    seed: int = 20160905
    n_thermalize: int = 500
    n_samples: int = 200
    quenched: bool = False
    fermion_bc: str = "periodic"


def hamiltonian(st):
    """H = kin + S_G + S_F (hmc.py:44-51)."""
    U = _links(st)
    return (kinetic_energy(st.p) + gauge_action(st.q, st.beta)
            + fermion_action(U, st.m0, st.eta, st.tol, st.counter, st.stop))


def metropolis(dh, rng):
    """hmc.py:54-60."""
    if not np.isfinite(dh):
        raise ValueError(f"non-finite energy change {dh}")
    if dh <= 0.0:
        return True
    return bool(rng.random() < np.exp(-dh))


def hmc_update(q, cfg, rng, counter=None):
    """One unbatched HMC update (hmc.py:69-95). Returns (q', dict)."""
    counter = counter if counter is not None else Counter()
    L, T = cfg.L, cfg.T
    p = sample_momenta(rng, L, T)
    if cfg.quenched:
        eta = np.zeros((L, T, 2), dtype=np.complex128)
    else:
        eta = pseudofermion_heatbath(fermion_links(q, cfg.fermion_bc), cfg.m0, rng, L, T)
    st = State(q.copy(), p, eta, cfg.beta, cfg.m0, cfg.cg_tol, counter, cfg.fermion_bc)
    h0 = hamiltonian(st)
    n, inv = integrate(st, cfg.scheme, cfg.h, cfg.tau, cfg.micro_per_call, cfg.micro_ratio)
    h1 = hamiltonian(st)
    dh = float(h1 - h0)
    acc = metropolis(dh, rng)
    return (st.q if acc else q), dict(dh=dh, accepted=acc, inversions=inv, n_steps=n)


def measure_dh(q0, cfg, rng, n_samples=None):
    """Batched fixed-start |dH| measurement, global CG stop (hmc.py:98-130)."""
    n = n_samples if n_samples is not None else cfg.n_samples
    L, T = cfg.L, cfg.T
    counter = Counter()
    p = sample_momenta(rng, L, T, batch=n)
    if cfg.quenched:
        eta = np.zeros((n, L, T, 2), dtype=np.complex128)
    else:
        eta = pseudofermion_heatbath(fermion_links(q0, cfg.fermion_bc), cfg.m0, rng, L, T, batch=n)
    q = np.broadcast_to(q0, (n,) + q0.shape).copy()
    st = State(q, p, eta, cfg.beta, cfg.m0, cfg.cg_tol, counter, cfg.fermion_bc)
    h0 = hamiltonian(st)
    nsteps, inv = integrate(st, cfg.scheme, cfg.h, cfg.tau, cfg.micro_per_call, cfg.micro_ratio)
    h1 = hamiltonian(st)
    dh = np.asarray(h1 - h0, dtype=np.float64)
    ad = np.abs(dh)
    return dict(dh=dh, mean_abs=float(ad.mean()),
                stderr=float(ad.std(ddof=1) / np.sqrt(n)) if n > 1 else 0.0,
                acceptance=float(np.mean(np.minimum(1.0, np.exp(-dh)))),
                inversions_per_traj=inv, n_steps=nsteps)


def thermalize(cfg, rng):
    """Cold start + annealed leapfrog updates (hmc.py:133-155)."""
    q = np.zeros((2, cfg.L, cfg.T))
    tc = replace(cfg, scheme="leapfrog", h=min(cfg.h, 0.1), micro_per_call=None)
    hits, hist = 0, []
    for i in range(cfg.n_thermalize):
        q, s = hmc_update(q, tc, rng)
        hits += s["accepted"]
        hist.append(float(avg_plaquette(q)))
        if (i + 1) % 20 == 0:
            if hits < 0.8 * 20:
                tc = replace(tc, h=tc.h * 0.7)
            hits = 0
    return q, hist


# ---------------------------------------------------------------------------
# ensemble helper: B independent chains, each exactly an unbatched hmc_update
# on its own stream (make_rng(seed, stream=chain)).
# ---------------------------------------------------------------------------

def ensemble_hot_start(cfg, n_chains, seed, stream0=0):
    rngs = [make_rng(seed, stream0 + c) for c in range(n_chains)]
    q = np.stack([hot_start(r, cfg.L, cfg.T) for r in rngs])
    return q, rngs


def ensemble_update(q, cfg, rngs):
    out, stats = [], []
    for c, rng in enumerate(rngs):
        qc, s = hmc_update(q[c], cfg, rng)
        out.append(qc)
        stats.append(s)
    return np.stack(out), stats
