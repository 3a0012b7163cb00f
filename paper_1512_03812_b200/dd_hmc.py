"""HMC trajectories on a domain-decomposed lattice (BASELINE configs[4]:
one 2048^2 lattice, adapted nested force-gradient).

Fields live as extended strips (dd.py).  Every elementary map of the
integrator programs (integrators.PROGRAMS) is implemented here with the
face exchanges it needs, so the same schedules drive both paths:

* drift           q <- wrap(q + dt p) on every row, then exchange q's faces
* kick_gauge      fused gauge force + kick (plaquettes need q one row out)
* kick_fermion /  xi = DD-CG(eta); chi = D xi (faces of xi exchanged first,
  kick_full       chi's afterwards); fused force + kick
* kick_fg_fermion force, weighted w-sums, Z1 = D CG(b1), Z2 = CG(D^dag(b2+Z1)),
                  force-gradient contraction — each stencil's input faces
                  exchanged first
* inner_leapfrog  micro steps with one q exchange after every drift
* Hamiltonian     whole-lattice sums of the own rows (sch_dd_own_sum: the
                  canonical tree, strip-count invariant)

* kick_fg_full     gauge force, fermion force, C_GG (plaquettes two rows
                  out: the 2-row halo), the gauge Hessian dot f and both
                  fermion Hessian dots (weights g and f, faces refreshed)
* kick_fg_approx  the force at q shifted along it (shifted links' faces
                  exchanged, a second chi/xi solve on them)
* inner_fg        micro 5-stage FG steps of the gauge action

All nine reference schemes run on strips.  With host draws scattered from
the full-lattice reference generator the result equals hmc_update on the
whole lattice (tests/test_gpu_dd.py).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .dd import DDWilsonDirac, StripLattice
from .fermion import InversionCounter, draw_phi
from .hmc import TrajectoryStats, metropolis
from .integrators import FG_KICK_SIGN, PROGRAMS, IntegratorSpec
from .lattice import LatticeGeom, NumpyDeviceRng, as_links, as_spinor

SUPPORTED = ("leapfrog", "5stage", "5stage-fg", "fg-approx", "11stage", "nested-leapfrog",
             "nested-5stage", "nested-fg", "adapted-nested-fg")


def _call(name, *args):
    _lib.ctx().call(name, *args)


@dataclass
class DDState:
    lat: StripLattice
    q: torch.Tensor      # (S, 2, Lext, T)
    p: torch.Tensor
    eta: torch.Tensor    # (S, Lext, T, 2)
    beta: float
    m0: float
    tol: float
    counter: InversionCounter
    fermion_bc: str = "periodic"
    _pair: tuple | None = None

    # -- geometry shortcuts -------------------------------------------------
    @property
    def S(self):
        return self.lat.S

    @property
    def Lext(self):
        return self.lat.Lext

    @property
    def T(self):
        return self.lat.T

    def xlinks(self, f):
        return self.lat.exchange(f, 2, 1)

    def xspin(self, f):
        return self.lat.exchange(f, 1, 4)

    # -- fermion pieces -------------------------------------------------------
    def operator(self) -> DDWilsonDirac:
        return DDWilsonDirac(self.lat, self.q, self.m0, self.fermion_bc)

    def dslash(self, op: DDWilsonDirac, psi, dagger: bool):
        """D psi on the own rows (psi's faces exchanged first), faces of the
        result exchanged afterwards."""
        self.xspin(psi)
        out = torch.empty_like(psi)
        _call("sch_dslash", _lib.ptr(op.U), 1, _lib.ptr(psi), _lib.ptr(out), self.S, self.Lext,
              self.T, self.m0, int(dagger))
        return self.xspin(out)

    def cg(self, op: DDWilsonDirac, b):
        x, _, _ = op.cg(b, self.tol)
        return self.xspin(x)

    def solve_pair(self):
        """(op, chi, xi) at the current links; solves shared while q, eta unchanged."""
        op = self.operator()
        if self._pair is not None and self._pair[0] is self.q and self._pair[1] is self.eta:
            self.counter.add(2)
            return (op,) + self._pair[2:]
        xi = self.cg(op, self.eta)
        chi = self.dslash(op, xi, False)
        self.counter.add(2)
        self._pair = (self.q, self.eta, chi, xi)
        return op, chi, xi


# ---------------------------------------------------------------------------
# elementary maps
# ---------------------------------------------------------------------------

def _drift(st: DDState, dt: float):
    out = torch.empty_like(st.q)
    _call("sch_rotate_links", _lib.ptr(st.q), _lib.ptr(st.p), float(dt), _lib.ptr(out), st.q.numel())
    st.q = st.xlinks(out)


def _kick_gauge(st: DDState, dt: float):
    if dt == 0.0:
        return
    out = torch.empty_like(st.p)
    _call("sch_kick_gauge", _lib.ptr(st.q), _lib.ptr(st.p), float(st.beta), float(dt), _lib.ptr(out),
          st.S, st.Lext, st.T)
    st.p = out


def _kick_fermion(st: DDState, dt: float, full: bool = False):
    if dt == 0.0:
        return
    op, chi, xi = st.solve_pair()
    out = torch.empty_like(st.p)
    _call("sch_kick_fermion", _lib.ptr(op.U), _lib.ptr(chi), _lib.ptr(xi),
          _lib.ptr(st.q) if full else None, float(st.beta), _lib.ptr(st.p), float(dt), _lib.ptr(out),
          st.S, st.Lext, st.T)
    st.p = out


def _fermion_force(st: DDState, op, chi, xi):
    """f on every row whose stencil stays inside the strip, faces refreshed
    (weights are read one row out of the own range)."""
    f = torch.empty_like(st.p)
    _call("sch_fermion_force", _lib.ptr(op.U), _lib.ptr(chi), _lib.ptr(xi), _lib.ptr(f), st.S,
          st.Lext, st.T)
    return st.xlinks(f)


def _gauge_force(st: DDState, q=None):
    """beta-scaled gauge force of q (default: the state's links), faces refreshed."""
    q = st.q if q is None else q
    g = torch.empty_like(q)
    _call("sch_gauge_force", _lib.ptr(q), float(st.beta), _lib.ptr(g), st.S, st.Lext, st.T)
    return st.xlinks(g)


def _fg_gauge_gauge(st: DDState):
    """C_GG: plaquettes up to two rows out of each own row, i.e. the 2-row halo."""
    out = torch.empty_like(st.q)
    _call("sch_fg_gauge_gauge", _lib.ptr(st.q), float(st.beta), _lib.ptr(out), st.S, st.Lext, st.T)
    return out


def _gauge_hessian_dot(st: DDState, w):
    out = torch.empty_like(st.q)
    _call("sch_gauge_hessian_dot", _lib.ptr(st.q), float(st.beta), _lib.ptr(w), _lib.ptr(out), st.S,
          st.Lext, st.T)
    return out


def _fermion_hessian_dot(st: DDState, op, chi, xi, weight):
    """fg_fermion_hessian_dot (fermion.py:397-417) on strips: weighted w-sums,
    Z1 = D^{-dag} b1, Z2 = D^{-1}(b2 + Z1), contraction; 2 inversions."""
    b1, b2 = torch.empty_like(chi), torch.empty_like(chi)
    _call("sch_weighted_w_sums", _lib.ptr(op.U), _lib.ptr(weight), _lib.ptr(chi), _lib.ptr(xi),
          _lib.ptr(b1), _lib.ptr(b2), st.S, st.Lext, st.T)
    z1 = st.dslash(op, st.cg(op, st.xspin(b1)), False)        # D^{-dag} b1
    st.counter.add(1)
    t = torch.empty_like(b2)
    _call("sch_kick", _lib.ptr(b2), _lib.ptr(z1), -1.0, None, 0.0, _lib.ptr(t), 2 * t.numel())
    z2 = st.cg(op, st.dslash(op, t, True))                    # D^{-1} (b2 + z1)
    st.counter.add(1)
    fg = torch.empty_like(st.p)
    _call("sch_fg_fermion_combine", _lib.ptr(op.U), _lib.ptr(z1), _lib.ptr(z2), _lib.ptr(chi),
          _lib.ptr(xi), _lib.ptr(weight), _lib.ptr(fg), st.S, st.Lext, st.T)
    return fg


def _fg_kick(st: DDState, force, b_dt: float, fg, c_dt3: float):
    out = torch.empty_like(st.p)
    _call("sch_kick", _lib.ptr(st.p), _lib.ptr(force), float(b_dt), _lib.ptr(fg),
          float(FG_KICK_SIGN * c_dt3), _lib.ptr(out), st.p.numel())
    st.p = out


def _kick_fg_fermion(st: DDState, b_dt: float, c_dt3: float):
    if c_dt3 == 0.0:
        _kick_fermion(st, b_dt)
        return
    op, chi, xi = st.solve_pair()
    f = _fermion_force(st, op, chi, xi)
    _fg_kick(st, f, b_dt, _fermion_hessian_dot(st, op, chi, xi, f), c_dt3)


def _kick_fg_full(st: DDState, b_dt: float, c_dt3: float):
    """integrators.kick_fg_full on strips; 6 inversions."""
    if c_dt3 == 0.0:
        _kick_fermion(st, b_dt, full=True)
        return
    op, chi, xi = st.solve_pair()
    f = _fermion_force(st, op, chi, xi)
    g = _gauge_force(st)
    fg = ((_fg_gauge_gauge(st) + _gauge_hessian_dot(st, f)) + _fermion_hessian_dot(st, op, chi, xi, g)) \
        + _fermion_hessian_dot(st, op, chi, xi, f)
    _fg_kick(st, g + f, b_dt, fg, c_dt3)


def _kick_fg_approx(st: DDState, b_dt: float, c_dt3: float):
    """integrators.kick_fg_approx on strips: the force at q shifted along the
    force; 4 inversions."""
    if c_dt3 == 0.0:
        _kick_fermion(st, b_dt, full=True)
        return
    op, chi, xi = st.solve_pair()
    force = _gauge_force(st) + _fermion_force(st, op, chi, xi)
    qs = torch.empty_like(st.q)
    _call("sch_rotate_links", _lib.ptr(st.q), _lib.ptr(force), float(2.0 * FG_KICK_SIGN * c_dt3 / b_dt),
          _lib.ptr(qs), qs.numel())
    qs = st.xlinks(qs)
    op2 = DDWilsonDirac(st.lat, qs, st.m0, st.fermion_bc)
    xi2 = st.cg(op2, st.eta)
    chi2 = st.dslash(op2, st.xspin(xi2), False)
    st.counter.add(2)
    shifted = _gauge_force(st, qs) + _fermion_force(st, op2, chi2, xi2)
    _fg_kick(st, shifted, b_dt, None, 0.0)


def _kick_fg_gauge(st: DDState, b_dt: float, c_dt3: float):
    if c_dt3 == 0.0:
        _kick_gauge(st, b_dt)
        return
    _fg_kick(st, _gauge_force(st), b_dt, _fg_gauge_gauge(st), c_dt3)


def _inner_fg(st: DDState, span: float, m: int, fgc: float):
    delta = span / m
    c_d3 = fgc * delta**3
    for _ in range(m):
        _kick_gauge(st, delta / 6.0)
        _drift(st, 0.5 * delta)
        _kick_fg_gauge(st, 2.0 * delta / 3.0, c_d3)
        _drift(st, 0.5 * delta)
        _kick_gauge(st, delta / 6.0)


def _inner_leapfrog(st: DDState, span: float, m: int):
    delta = span / m
    for _ in range(m):
        _kick_gauge(st, 0.5 * delta)
        _drift(st, delta)
        _kick_gauge(st, 0.5 * delta)


def _run_program(st: DDState, scheme: str, h: float, m: int, fgc: float):
    for name, weight in PROGRAMS[scheme]:
        w = weight(h)
        if name == "D":
            _drift(st, w)
        elif name == "K":
            _kick_fermion(st, w, full=True)
        elif name == "Kf":
            _kick_fermion(st, w)
        elif name == "Gfermion":
            _kick_fg_fermion(st, w, fgc * h**3)
        elif name == "Gfull":
            _kick_fg_full(st, w, fgc * h**3)
        elif name == "Gapprox":
            _kick_fg_approx(st, w, fgc * h**3)
        elif name == "Ileapfrog":
            _inner_leapfrog(st, w, m)
        elif name == "Ifg":
            _inner_fg(st, w, m, fgc)
        else:
            raise NotImplementedError(f"{name} in {scheme} is not wired for strips")


def dd_hamiltonian(st: DDState) -> float:
    """H = kin + S_G + S_F over the whole lattice (hmc.py:44-51).  Each sum is
    formed on the device by the lattice's canonical tree through its
    transport (sch_dd_own_sum), so every rank gets the same bits for any
    number of strips; one host read for the three."""
    _, _, xi = st.solve_pair()
    out = torch.empty((3,), dtype=torch.float64, device=st.q.device)
    _call("sch_dd_own_sum", st.lat._handle, 0, _lib.ptr(st.p), None, _lib.ptr(out[0:1]))
    _call("sch_dd_own_sum", st.lat._handle, 1, _lib.ptr(st.q), None, _lib.ptr(out[1:2]))
    _call("sch_dd_own_sum", st.lat._handle, 2, _lib.ptr(st.eta), _lib.ptr(xi), _lib.ptr(out[2:3]))
    psq, gsum, s_f = out.tolist()
    return (0.5 * psq + st.beta * gsum) + s_f


def dd_integrate(st: DDState, spec: IntegratorSpec, tau: float):
    if spec.scheme not in SUPPORTED:
        raise NotImplementedError(f"scheme {spec.scheme!r} on strips: supported {SUPPORTED}")
    n_steps = max(1, round(tau / spec.h))
    before = st.counter.count
    for _ in range(n_steps):
        _run_program(st, spec.scheme, spec.h, spec.micro_steps(), spec.fg_coefficient)
    return n_steps, st.counter.count - before


def dd_hmc_update(lat: StripLattice, q_ext, config, rng):
    """One HMC update of the decomposed lattice, drawing in the reference
    order from the full-lattice generator ``rng`` (hmc.py:69-95).  Returns
    (links, TrajectoryStats); on reject the caller's links come back.

    ``rng`` is a host ``np.random.Generator`` or a one-stream
    ``NumpyDeviceRng``: the device generator walks the same Philox/ziggurat
    stream on the GPU (csrc/nprng.cu), so every rank draws the whole-lattice
    p and phi there and keeps its own rows — the same values as the host
    draws, no host generation or upload."""
    L, T = config.L, config.T
    device_rng = isinstance(rng, NumpyDeviceRng)
    if device_rng:
        if rng.n != 1:
            raise ValueError(f"the decomposed lattice draws one stream, got {rng.n}")
        p_dev, phi_dev = rng.heatbath(LatticeGeom(L, T), quenched=config.quenched)
        p_full = p_dev[0]
        phi_full = None if phi_dev is None else phi_dev[0]
    else:
        p_full = rng.standard_normal((2, L, T))
        phi_full = None if config.quenched else draw_phi(rng, L, T)
    q_in = as_links(q_ext)
    q0 = lat.exchange(q_in.clone(), 2, 1)
    st = DDState(lat, q0, lat.scatter_links(p_full),
                 torch.zeros((lat.S, lat.Lext, T, 2), dtype=torch.complex128, device=q0.device),
                 config.beta, config.m0, config.cg_tol, InversionCounter(), config.fermion_bc)
    if phi_full is not None:
        st.eta = st.dslash(st.operator(), lat.scatter_spinor(phi_full), True)
    h_start = dd_hamiltonian(st)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    spec = IntegratorSpec(config.scheme, config.h, micro_per_call=config.micro_per_call,
                          micro_ratio=config.micro_ratio)
    n_steps, inv = dd_integrate(st, spec, config.tau)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    h_end = dd_hamiltonian(st)
    dh = float(h_end - h_start)
    if device_rng:   # hmc.py:54-60 on the device stream (one uniform iff dH > 0)
        flag = int(rng.metropolis(torch.tensor([dh], dtype=torch.float64,
                                               device=st.q.device)).item())
        if flag < 0:
            raise ValueError(f"non-finite energy change dH={dh}")
        accepted = bool(flag)
    else:
        accepted = metropolis(dh, rng)
    stats = TrajectoryStats(dh=dh, accepted=accepted, inversions=inv, n_steps=n_steps,
                            wall_time=wall)
    return (st.q if accepted else q_ext), stats
