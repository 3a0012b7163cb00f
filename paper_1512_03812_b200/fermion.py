"""Wilson fermions on the B200: D / D^dag / D^dag D, batched CG with the
reference's exact stopping rule, pseudofermion heatbath and action, chi/xi
solves, the fermion force and the fermion force-gradient pieces.

Mirror of ``schwinger.fermion`` (pkg/src/schwinger/fermion.py).  The
signatures, inversion accounting and error behaviour are the reference's;
``stop=`` is the one addition ("batch_global" = the reference's batched
semantics, "per_chain" = one unbatched reference call per chain, used by the
chain ensemble).  Every operator launches sm_100a kernels through the C-ABI.

Reports are lazy: ``SolveReport.iterations`` / ``rel_residual`` synchronise
with the device only when read, so the integrators never stall on them.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .lattice import as_links, as_spinor, geom_of, kick, n_chains, squeeze_chain

DEFAULT_TOL = 1e-12          # fermion.py:28
DEFAULT_MAXITER = 10_000     # fermion.py:29

STOP_MODES = {"batch_global": 0, "per_chain": 1}
FERMION_BC = {"periodic": 0, "antiperiodic": 1}


class SolverError(RuntimeError):
    """CG hit its iteration cap (fermion.py:63-68)."""

    def __init__(self, message, best_residual):
        super().__init__(f"{message} (best relative residual {best_residual:.3e})")
        self.best_residual = best_residual


class InversionCounter:
    """Monotonic tally of Dirac inversions (fermion.py:71-78)."""

    def __init__(self):
        self.count = 0

    def add(self, n: int):
        self.count += n


class CgInfo:
    """Per-chain CG outcome kept on the device until someone asks."""

    def __init__(self, iters: torch.Tensor, relres: torch.Tensor, status: torch.Tensor,
                 batched: bool, stop: str, maxiter: int):
        self.iters_dev, self.relres_dev, self.status_dev = iters, relres, status
        self.batched, self.stop, self.maxiter = batched, stop, maxiter

    def iterations(self):
        it = self.iters_dev.cpu().numpy()
        if not self.batched or self.stop == "batch_global":
            return int(it.max())
        return it.astype(np.int64)

    def worst_rel(self) -> float:
        return float(self.relres_dev.max().item())

    def raise_if_failed(self):
        st = self.status_dev.cpu().numpy()
        if st.any():
            rel = self.relres_dev.cpu().numpy()[st != 0]
            raise SolverError(f"CG exceeded {self.maxiter} iterations", float(rel.max()))


class SolveReport:
    """(iterations, rel_residual, inversions) of one solve (fermion.py:81-85),
    evaluated lazily from the device."""

    def __init__(self, inversions: int, info: CgInfo | None = None, iterations: int | None = None,
                 rel_fn=None):
        self.inversions = inversions
        self._info = info
        self._iterations = iterations
        self._rel_fn = rel_fn
        self._rel = None

    @property
    def iterations(self):
        if self._iterations is None:
            it = self._info.iterations()
            self._iterations = int(np.max(it))
        return self._iterations

    @property
    def rel_residual(self) -> float:
        if self._rel is None:
            self._rel = float(self._rel_fn()) if self._rel_fn is not None else self._info.worst_rel()
        return self._rel

    def __repr__(self):
        return (f"SolveReport(iterations={self.iterations}, rel_residual={self.rel_residual:.3e}, "
                f"inversions={self.inversions})")


def _spinor_batch(psi: torch.Tensor) -> int:
    return n_chains(psi, 3)


class WilsonDirac:
    """Wilson-Dirac operator bound to one (batched) gauge configuration
    (fermion.py:88-160).  ``U = exp(i q)`` is built by the link-cache kernel;
    ``fermion_bc='antiperiodic'`` flips the time links on the last slice
    (BASELINE configs; the reference itself is periodic, fermion.py:11)."""

    def __init__(self, q, m0: float, fermion_bc: str = "periodic"):
        self.q = as_links(q)
        self.m0 = float(m0)
        self.fermion_bc = fermion_bc
        g = geom_of(self.q)
        self.L, self.T = g.L, g.T
        self.B = n_chains(self.q)
        self.U = torch.empty(self.q.shape, dtype=torch.complex128, device=self.q.device)
        _lib.ctx().call("sch_links_to_u", _lib.ptr(self.q), _lib.ptr(self.U), self.B, self.L,
                        self.T, FERMION_BC[fermion_bc])
        self._dense = None
        self._u_cache = {}

    @property
    def geom_shape(self):
        return (self.L, self.T)

    @property
    def batch_shape(self):
        return tuple(self.q.shape[:-3])

    # -- broadcasting between the link batch and the spinor batch ----------
    def _U_for(self, batch_shape) -> torch.Tensor:
        if tuple(batch_shape) == self.batch_shape:
            return self.U
        key = tuple(batch_shape)
        if key not in self._u_cache:
            self._u_cache[key] = self.U.expand(key + tuple(self.U.shape[-3:])).contiguous()
        return self._u_cache[key]

    def _prep(self, psi):
        psi = as_spinor(psi)
        if tuple(psi.shape[-3:]) != (self.L, self.T, 2):
            raise ValueError(f"spinor shape {tuple(psi.shape)} does not match lattice {self.L}x{self.T}")
        bshape = torch.broadcast_shapes(tuple(psi.shape[:-3]), self.batch_shape)
        if tuple(psi.shape[:-3]) != tuple(bshape):
            psi = psi.expand(tuple(bshape) + (self.L, self.T, 2)).contiguous()
        return psi, tuple(bshape)

    def _dslash(self, psi, dagger: bool):
        psi, bshape = self._prep(psi)
        B = n_chains(psi)
        out = torch.empty_like(psi)
        if self.batch_shape == bshape:
            U, ub = self.U, 1
        elif self.B == 1:
            U, ub = self.U, 0
        else:
            U, ub = self._U_for(bshape), 1
        _lib.ctx().call("sch_dslash", _lib.ptr(U), ub, _lib.ptr(psi), _lib.ptr(out), B, self.L,
                        self.T, self.m0, int(dagger))
        return out

    def apply(self, psi) -> torch.Tensor:
        """D psi (fermion.py:119-122); kernel k_dslash<false>."""
        return self._dslash(psi, False)

    def apply_dag(self, psi) -> torch.Tensor:
        """D^dag psi (fermion.py:124-127); kernel k_dslash<true>."""
        return self._dslash(psi, True)

    def normal(self, psi) -> torch.Tensor:
        """D^dag D psi in one fused shared-memory tile pass (fermion.py:129-131)."""
        psi, bshape = self._prep(psi)
        U = self._U_for(bshape)
        out = torch.empty_like(psi)
        _lib.ctx().call("sch_ddagd", _lib.ptr(U), _lib.ptr(psi), _lib.ptr(out), n_chains(psi),
                        self.L, self.T, self.m0)
        return out

    # -- dense path for tiny lattices (fermion.py:133-160; test mode only) --
    def dense_matrix(self) -> torch.Tensor:
        """D as a (2V, 2V) matrix, built by applying the GPU operator to basis
        vectors (all 2V columns in one batched launch)."""
        if self.q.ndim != 3:
            raise ValueError("dense path needs an unbatched configuration")
        dim = 2 * self.L * self.T
        basis = torch.eye(dim, dtype=torch.complex128, device=self.q.device)
        cols = self._dslash(basis.reshape(dim, self.L, self.T, 2), False)
        return cols.reshape(dim, dim).T.contiguous()

    def _dense_normal(self):
        if self._dense is None:
            d = self.dense_matrix()
            self._dense = (d, d.conj().T @ d)
        return self._dense

    def solve_normal_dense(self, b) -> torch.Tensor:
        """Exact (D^dag D)^{-1} b via a dense LU (test-mode ``exact_solves``)."""
        b = as_spinor(b)
        _, ndag = self._dense_normal()
        flat = b.reshape(b.shape[:-3] + (-1,))
        x = torch.linalg.solve(ndag, flat.unsqueeze(-1)).squeeze(-1)
        return x.reshape(b.shape)


# ---------------------------------------------------------------------------
# inner products
# ---------------------------------------------------------------------------

def spinor_dot(a, b) -> torch.Tensor:
    """sum conj(a) b over sites and spin per chain (fermion.py:54-56)."""
    a, b = as_spinor(a), as_spinor(b)
    if a.shape != b.shape:
        shape = torch.broadcast_shapes(a.shape, b.shape)
        a, b = a.expand(shape).contiguous(), b.expand(shape).contiguous()
    B = n_chains(a)
    out = torch.empty((B,), dtype=torch.complex128, device=a.device)
    _lib.ctx().call("sch_spinor_dot", _lib.ptr(a), _lib.ptr(b), _lib.ptr(out), B,
                    a.numel() // (2 * B))
    return squeeze_chain(out, a)


def spinor_norm(a) -> torch.Tensor:
    return torch.sqrt(spinor_dot(a, a).real)


# ---------------------------------------------------------------------------
# conjugate gradient on the normal equations (fermion.py:171-217)
# ---------------------------------------------------------------------------

# When set to a list, every cg_solve appends (start_event, end_event,
# iters_tensor, sites_per_chain) so a benchmark can time the CG kernels on
# their own stream and count the iterations they ran.  Inside a CUDA-graph
# capture the events are external event-record nodes: after each replay
# they hold that replay's timestamps (and the iteration tensors its counts).
CG_PROFILE: list | None = None


def _profile_events():
    ext = torch.cuda.is_current_stream_capturing()
    return (torch.cuda.Event(enable_timing=True, external=ext),
            torch.cuda.Event(enable_timing=True, external=ext))


def cg_solve(op: WilsonDirac, b, tol: float, maxiter: int = DEFAULT_MAXITER, x0=None,
             stop: str = "batch_global"):
    """Device-side CG; returns (x, CgInfo) without synchronising."""
    b, bshape = op._prep(b)
    U = op._U_for(bshape)
    B = n_chains(b)
    x = torch.empty_like(b)
    if x0 is not None:
        x0 = as_spinor(x0).expand(b.shape).contiguous()
    dev = b.device
    iters = torch.empty((B,), dtype=torch.int32, device=dev)
    relres = torch.empty((B,), dtype=torch.float64, device=dev)
    status = torch.empty((B,), dtype=torch.int32, device=dev)
    prof = CG_PROFILE
    if prof is not None:
        ev0, ev1 = _profile_events()
        ev0.record()
    _lib.ctx().call("sch_cg_normal", _lib.ptr(U), _lib.ptr(b), _lib.ptr(x), _lib.ptr(x0), B, op.L,
                    op.T, op.m0, float(tol), int(maxiter), STOP_MODES[stop], _lib.ptr(iters),
                    _lib.ptr(relres), _lib.ptr(status), None)
    if prof is not None:
        ev1.record()
        prof.append((ev0, ev1, iters, op.L * op.T))
    return x, CgInfo(iters, relres, status, len(bshape) > 0, stop, maxiter)


def cg_normal(op: WilsonDirac, b, tol: float, maxiter: int = DEFAULT_MAXITER, x0=None,
              stop: str = "batch_global"):
    """CG for (D^dag D) x = b with the reference's stopping rule; returns
    (x, iterations, worst relative residual) and raises SolverError at the
    cap (fermion.py:171-217)."""
    x, info = cg_solve(op, b, tol, maxiter, x0, stop)
    info.raise_if_failed()
    return x, info.iterations(), info.worst_rel()


def _rel_residual(residual, b) -> float:
    nb = spinor_norm(b).reshape(-1)
    nr = spinor_norm(residual).reshape(-1)
    safe = torch.where(nb > 0, nb, torch.ones_like(nb))
    return float(torch.where(nb > 0, nr / safe, torch.zeros_like(nb)).max().item())


def solve_normal(op: WilsonDirac, b, tol: float = DEFAULT_TOL, counter: InversionCounter | None = None,
                 x0=None, maxiter: int = DEFAULT_MAXITER, exact: bool = False,
                 stop: str = "batch_global", check: bool = True):
    """x = (D^dag D)^{-1} b; two inversions (fermion.py:233-242)."""
    if exact:
        x = op.solve_normal_dense(b)
        rep = SolveReport(2, iterations=0, rel_fn=lambda: _rel_residual(b - op.normal(x), b))
    else:
        x, info = cg_solve(op, b, tol, maxiter, x0, stop)
        if check:
            info.raise_if_failed()
        rep = SolveReport(2, info)
    if counter is not None:
        counter.add(2)
    return x, rep


def solve_dirac(op: WilsonDirac, b, tol: float = DEFAULT_TOL, counter: InversionCounter | None = None,
                x0=None, maxiter: int = DEFAULT_MAXITER, exact: bool = False,
                stop: str = "batch_global", check: bool = True):
    """x = D^{-1} b = CG(D^dag D, D^dag b); one inversion (fermion.py:245-259)."""
    rhs = op.apply_dag(b)
    if exact:
        x, info = op.solve_normal_dense(rhs), None
    else:
        x, info = cg_solve(op, rhs, tol, maxiter, x0, stop)
        if check:
            info.raise_if_failed()
    if counter is not None:
        counter.add(1)
    rep = SolveReport(1, info, iterations=0 if exact else None,
                      rel_fn=lambda: _rel_residual(as_spinor(b) - op.apply(x), b))
    return x, rep


def solve_dirac_dagger(op: WilsonDirac, b, tol: float = DEFAULT_TOL,
                       counter: InversionCounter | None = None, x0=None,
                       maxiter: int = DEFAULT_MAXITER, exact: bool = False,
                       stop: str = "batch_global", check: bool = True):
    """x = D^{-dag} b = D CG(D^dag D, b); one inversion (fermion.py:262-276)."""
    if exact:
        y, info = op.solve_normal_dense(b), None
        x = op.apply(y)
    else:   # one call: the resident engines apply D inside the solve
        x, y, info = _solve_apply(op, b, tol, maxiter, x0, stop)
        if check:
            info.raise_if_failed()
    if counter is not None:
        counter.add(1)
    rep = SolveReport(1, info, iterations=0 if exact else None,
                      rel_fn=lambda: _rel_residual(as_spinor(b) - op.apply_dag(x), b))
    return x, rep


# ---------------------------------------------------------------------------
# pseudofermions (fermion.py:283-310)
# ---------------------------------------------------------------------------

def draw_phi(rng, L: int, T: int, batch: int | None = None) -> np.ndarray:
    """phi = (N + iN)/sqrt(2) drawn with the reference generator, real part
    first (fermion.py:289)."""
    shape = (L, T, 2) if batch is None else (batch, L, T, 2)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)


def pseudofermion_heatbath(op: WilsonDirac, rng, batch: int | None = None) -> torch.Tensor:
    """eta = D^dag phi (fermion.py:283-290); phi from the host generator, or
    from a ``DeviceRng`` (bench mode) when one is passed."""
    from .lattice import DeviceRng

    if isinstance(rng, DeviceRng):
        nb = batch if batch is not None else 1
        phi = rng.complex_normal(nb, (op.L, op.T, 2), 1.0 / np.sqrt(2.0))
        if batch is None:
            phi = phi[0]
        return op.apply_dag(phi)
    return op.apply_dag(draw_phi(rng, op.L, op.T, batch))


def fermion_action(op: WilsonDirac, eta, tol: float = DEFAULT_TOL,
                   counter: InversionCounter | None = None, exact: bool = False,
                   stop: str = "batch_global") -> torch.Tensor:
    """S_F = Re <eta, (D^dag D)^{-1} eta> per chain; one normal solve (fermion.py:293-297)."""
    x, _ = solve_normal(op, eta, tol, counter=counter, exact=exact, stop=stop)
    return spinor_dot(eta, x).real


def _solve_apply(op: WilsonDirac, b, tol: float, maxiter: int, x0, stop: str):
    """(D x, x, CgInfo) for x = CG(D^dag D, b) in one C call (sch_chi_xi)."""
    b, bshape = op._prep(b)
    U = op._U_for(bshape)
    B = n_chains(b)
    x, dx = torch.empty_like(b), torch.empty_like(b)
    if x0 is not None:
        x0 = as_spinor(x0).expand(b.shape).contiguous()
    dev = b.device
    iters = torch.empty((B,), dtype=torch.int32, device=dev)
    relres = torch.empty((B,), dtype=torch.float64, device=dev)
    status = torch.empty((B,), dtype=torch.int32, device=dev)
    prof = CG_PROFILE
    if prof is not None:
        ev0, ev1 = _profile_events()
        ev0.record()
    _lib.ctx().call("sch_chi_xi", _lib.ptr(U), _lib.ptr(b), _lib.ptr(dx), _lib.ptr(x),
                    _lib.ptr(x0), B, op.L, op.T, op.m0, float(tol), int(maxiter),
                    STOP_MODES[stop], _lib.ptr(iters), _lib.ptr(relres), _lib.ptr(status))
    if prof is not None:
        ev1.record()
        prof.append((ev0, ev1, iters, op.L * op.T))
    return dx, x, CgInfo(iters, relres, status, len(bshape) > 0, stop, maxiter)


def chi_xi(op: WilsonDirac, eta, tol: float = DEFAULT_TOL, counter: InversionCounter | None = None,
           x0=None, exact: bool = False, stop: str = "batch_global", check: bool = True):
    """xi = (D^dag D)^{-1} eta, chi = D xi; two inversions (fermion.py:300-310).
    One C call (sch_chi_xi): the resident engines form chi inside the solve."""
    if exact:
        xi, report = solve_normal(op, eta, tol, counter=counter, x0=x0, exact=True, stop=stop,
                                  check=check)
        return op.apply(xi), xi, report
    chi, xi, info = _solve_apply(op, eta, tol, DEFAULT_MAXITER, x0, stop)
    if check:
        info.raise_if_failed()
    if counter is not None:
        counter.add(2)
    return chi, xi, SolveReport(2, info)


# ---------------------------------------------------------------------------
# force and force-gradient building blocks (fermion.py:317-439)
# ---------------------------------------------------------------------------

def _link_out(op: WilsonDirac, like: torch.Tensor) -> torch.Tensor:
    return torch.empty(like.shape[:-3] + (2, op.L, op.T), dtype=torch.float64, device=like.device)


def _spinors(op, *fields):
    out = [op._prep(f)[0] for f in fields]
    shape = torch.broadcast_shapes(*(f.shape for f in out))
    return [f.expand(shape).contiguous() if f.shape != shape else f for f in out]


def link_bilinears(op: WilsonDirac, mu: int, a, b):
    """The two hopping contractions attached to link (n, mu) (fermion.py:317-327):
    A(n) = a(n)^dag (1 - s_mu) U_mu(n) b(n + mu), B(n) = a(n + mu)^dag (1 + s_mu) U*_mu(n) b(n),
    as complex fields of shape a.shape[:-1]; kernel k_link_bilinears."""
    if mu not in (0, 1):
        raise ValueError(f"direction must be 0 or 1, got {mu}")
    a, b = _spinors(op, a, b)
    U = op._U_for(tuple(a.shape[:-3]))
    A = torch.empty(a.shape[:-1], dtype=torch.complex128, device=a.device)
    Bv = torch.empty_like(A)
    _lib.ctx().call("sch_link_bilinears", _lib.ptr(U), _lib.ptr(a), _lib.ptr(b), int(mu), _lib.ptr(A),
                    _lib.ptr(Bv), n_chains(a), op.L, op.T)
    return A, Bv


def fermion_force(op: WilsonDirac, chi, xi) -> torch.Tensor:
    """f(n,mu) = -Im[A - B] (fermion.py:330-336); kernel k_fermion_force."""
    chi, xi = _spinors(op, chi, xi)
    out = _link_out(op, chi)
    U = op._U_for(tuple(chi.shape[:-3]))
    _lib.ctx().call("sch_fermion_force", _lib.ptr(U), _lib.ptr(chi), _lib.ptr(xi), _lib.ptr(out),
                    n_chains(chi), op.L, op.T)
    return out


def kick_fermion_fused(op: WilsonDirac, chi, xi, p: torch.Tensor, dt: float, q=None,
                       beta: float = 0.0) -> torch.Tensor:
    """p - dt*f (kick_fermion) or p - dt*(beta*g(q) + f) (kick_full), one pass
    (integrators.py:172-186)."""
    out = torch.empty_like(p)
    _lib.ctx().call("sch_kick_fermion", _lib.ptr(op.U), _lib.ptr(chi), _lib.ptr(xi), _lib.ptr(q),
                    float(beta), _lib.ptr(p), float(dt), _lib.ptr(out), n_chains(p), op.L, op.T)
    return out


def weighted_w_sums(op: WilsonDirac, weight, chi, xi):
    """Aggregated derivative stencils b1 = sum weight*w1, b2 = sum weight*w2
    (fermion.py:362-383); kernel k_wsums."""
    chi, xi = _spinors(op, chi, xi)
    weight = as_links(weight).expand(chi.shape[:-3] + (2, op.L, op.T)).contiguous()
    b1, b2 = torch.empty_like(chi), torch.empty_like(chi)
    U = op._U_for(tuple(chi.shape[:-3]))
    _lib.ctx().call("sch_weighted_w_sums", _lib.ptr(U), _lib.ptr(weight), _lib.ptr(chi),
                    _lib.ptr(xi), _lib.ptr(b1), _lib.ptr(b2), n_chains(chi), op.L, op.T)
    return b1, b2


def z_pair(op: WilsonDirac, weight, chi, xi, tol: float = DEFAULT_TOL,
           counter: InversionCounter | None = None, exact: bool = False,
           stop: str = "batch_global", check: bool = True, infos: list | None = None):
    """Z1 = D^{-dag} b1, Z2 = D^{-1}(b2 + Z1); two inversions (fermion.py:386-394)."""
    b1, b2 = weighted_w_sums(op, weight, chi, xi)
    z1, r1 = solve_dirac_dagger(op, b1, tol, counter=counter, exact=exact, stop=stop, check=check)
    # b2 + Z1 on our kick kernel over the real view: b2 - (-1*Z1) == b2 + Z1 exactly
    b2z1 = torch.view_as_complex(kick(torch.view_as_real(b2), torch.view_as_real(z1), -1.0))
    z2, r2 = solve_dirac(op, b2z1, tol, counter=counter, exact=exact, stop=stop, check=check)
    if infos is not None:
        infos.extend(r._info for r in (r1, r2) if r._info is not None)
    return z1, z2


def fg_fermion_hessian_dot(op: WilsonDirac, chi, xi, weight, tol: float = DEFAULT_TOL,
                           counter: InversionCounter | None = None, exact: bool = False,
                           stop: str = "batch_global", check: bool = True,
                           infos: list | None = None) -> torch.Tensor:
    """2 * sum weight * Hess(S_F) via the Z trick (fermion.py:397-417);
    kernel k_fg_combine after the two Z solves."""
    chi, xi = _spinors(op, chi, xi)
    weight = as_links(weight).expand(chi.shape[:-3] + (2, op.L, op.T)).contiguous()
    z1, z2 = z_pair(op, weight, chi, xi, tol, counter=counter, exact=exact, stop=stop, check=check,
                    infos=infos)
    out = _link_out(op, chi)
    U = op._U_for(tuple(chi.shape[:-3]))
    _lib.ctx().call("sch_fg_fermion_combine", _lib.ptr(U), _lib.ptr(z1), _lib.ptr(z2), _lib.ptr(chi),
                    _lib.ptr(xi), _lib.ptr(weight), _lib.ptr(out), n_chains(chi), op.L, op.T)
    return out


def fg_fermion_fermion(op: WilsonDirac, eta, tol: float = DEFAULT_TOL,
                       counter: InversionCounter | None = None, exact: bool = False,
                       stop: str = "batch_global") -> torch.Tensor:
    """Fermion-fermion force-gradient piece from scratch (fermion.py:420-426)."""
    chi, xi, _ = chi_xi(op, eta, tol, counter=counter, exact=exact, stop=stop)
    f = fermion_force(op, chi, xi)
    return fg_fermion_hessian_dot(op, chi, xi, f, tol, counter=counter, exact=exact, stop=stop)


def fg_gauge_fermion(op: WilsonDirac, eta, beta: float, tol: float = DEFAULT_TOL,
                     counter: InversionCounter | None = None, exact: bool = False,
                     stop: str = "batch_global") -> torch.Tensor:
    """Fermion Hessian contracted with the gauge force (fermion.py:429-439)."""
    from .gauge import gauge_force

    chi, xi, _ = chi_xi(op, eta, tol, counter=counter, exact=exact, stop=stop)
    return fg_fermion_hessian_dot(op, chi, xi, gauge_force(op.q, beta), tol, counter=counter,
                                  exact=exact, stop=stop)
