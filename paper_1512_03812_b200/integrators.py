"""Reversible, volume-preserving MD integrators driving the B200 kernels.

Mirror of ``schwinger.integrators`` (pkg/src/schwinger/integrators.py): same
scheme ids, inversion accounting (INVERSIONS_PER_STEP), kick/drift/FG-kick
semantics and coefficient arithmetic.  Each scheme is written below as a
*program*: a palindromic list of elementary maps with their step weights,
interpreted by ``_make_step``.  The elementary maps call fused sm_100a
kernels (fermion-force+kick, gauge-force+kick, the resident inner-leapfrog
kernel, the CG engines).

B200-side additions (all bit-identical to the reference schedule):
  * ``MdState.stop``: "per_chain" for chain ensembles (each chain's CG stops
    as an unbatched reference call would), "batch_global" otherwise.
  * ``MdState.reuse_solves``: the chi/xi pair depends only on (q, eta), so a
    kick_fermion right after another solve at the same q (FSAL across macro
    steps, and the Hamiltonian at either end of a trajectory) reuses it.  The
    inversion counter still follows the reference convention.
  * solver failures are collected on the device and raised as SolverError at
    the end of the trajectory (one host sync instead of one per solve).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import _lib
from .fermion import (InversionCounter, WilsonDirac, chi_xi, fermion_force,
                      fg_fermion_hessian_dot, kick_fermion_fused, SolverError)
from .gauge import fg_gauge_gauge, gauge_force, gauge_hessian_dot, kick_gauge_fused
from .lattice import as_links, geom_of, kick, n_chains, rotate_links

FG_KICK_SIGN = -1.0           # integrators.py:30
DEFAULT_FG_COEFF = 1.0 / 72.0  # integrators.py:32

# 11-stage composition point (integrators.py:40-43)
ELEVEN_SIGMA = 0.08398315262876693
ELEVEN_ETA = 0.2539785108410595
ELEVEN_LAM = 0.6822365335719091
ELEVEN_THETA = -0.03230286765269967


def fourth_order_defect(sigma: float, eta: float, lam: float, theta: float):
    """The two third-order error coefficients of the 11-stage palindrome
    (integrators.py:46-58); both vanish at a fourth-order point."""
    s, e, l, t = sigma, eta, lam, theta
    c1 = (12*e**2*s - 6*e**2 + 24*e*l*t + 24*e*s*t - 12*e*s - 12*e*t + 6*e
          + 12*l*t**2 - 12*l*t + 12*s*t**2 - 12*s*t - 6*t**2 + 6*t - 1) / 6.0
    c2 = (24*e*s**2 - 24*e*s + 6*e + 24*l**2*t + 48*l*s*t - 24*l*t
          + 24*s**2*t - 24*s*t + 6*t - 1) / 12.0
    return c1, c2


SCHEME_IDS = ("leapfrog", "5stage", "5stage-fg", "fg-approx", "11stage",
              "nested-leapfrog", "nested-5stage", "nested-fg", "adapted-nested-fg")
NESTED_SCHEMES = ("nested-leapfrog", "nested-5stage", "nested-fg", "adapted-nested-fg")
INVERSIONS_PER_STEP = {"leapfrog": 4, "5stage": 6, "5stage-fg": 10, "fg-approx": 8,
                       "11stage": 12, "nested-leapfrog": 4, "nested-5stage": 6,
                       "nested-fg": 8, "adapted-nested-fg": 8}


@dataclass
class MdState:
    """Links, momenta and the frozen pseudofermion on the device
    (integrators.py:82-104)."""

    q: torch.Tensor
    p: torch.Tensor
    eta: torch.Tensor
    beta: float
    m0: float
    tol: float = 1e-12
    counter: InversionCounter = field(default_factory=InversionCounter)
    exact_solves: bool = False
    fermion_bc: str = "periodic"
    stop: str = "batch_global"
    reuse_solves: bool = True
    _op: tuple | None = field(default=None, repr=False)
    _pair: tuple | None = field(default=None, repr=False)
    _infos: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        from .lattice import as_spinor
        self.q = as_links(self.q)
        self.p = as_links(self.p)
        self.eta = as_spinor(self.eta)

    def copy(self) -> "MdState":
        return MdState(self.q.clone(), self.p.clone(), self.eta.clone(), self.beta, self.m0,
                       self.tol, self.counter, self.exact_solves, self.fermion_bc, self.stop,
                       self.reuse_solves)

    def flip_momenta(self):
        self.p = kick(torch.zeros_like(self.p), self.p, 1.0)   # 0 - 1*p = -p exactly

    # -- device-side helpers ---------------------------------------------
    def operator(self) -> WilsonDirac:
        """WilsonDirac at the current links, cached while q is unchanged."""
        if self._op is None or self._op[0] is not self.q:
            self._op = (self.q, WilsonDirac(self.q, self.m0, self.fermion_bc))
        return self._op[1]

    def solve_pair(self):
        """(op, chi, xi) at the current (q, eta); two inversions counted."""
        op = self.operator()
        if (self.reuse_solves and not self.exact_solves and self._pair is not None
                and self._pair[0] is self.q and self._pair[1] is self.eta):
            self.counter.add(2)
            return op, self._pair[2], self._pair[3]
        chi, xi, rep = chi_xi(op, self.eta, self.tol, counter=self.counter,
                              exact=self.exact_solves, stop=self.stop, check=False)
        if rep._info is not None:
            self._infos.append(rep._info)
        self._pair = (self.q, self.eta, chi, xi)
        return op, chi, xi

    def check_solves(self):
        """Raise SolverError for any CG that hit its cap since the last check."""
        infos, self._infos = self._infos, []
        if not infos:
            return
        bad = torch.cat([i.status_dev.reshape(-1) for i in infos]).ne(0).any()   # 3 launches
        if bool(bad.item()):
            for i in infos:
                i.raise_if_failed()


@dataclass(frozen=True)
class IntegratorSpec:
    """Scheme and step sizes (integrators.py:107-143)."""

    scheme: str
    h: float
    micro_per_call: int | None = None
    micro_ratio: float = 10.0
    fg_coefficient: float = DEFAULT_FG_COEFF

    def __post_init__(self):
        if self.scheme not in SCHEME_IDS:
            raise ValueError(f"unknown scheme {self.scheme!r}; valid: {', '.join(SCHEME_IDS)}")
        if not self.h > 0:
            raise ValueError(f"step size must be positive, got {self.h}")
        if self.micro_per_call is not None and self.micro_per_call < 1:
            raise ValueError("micro_per_call must be >= 1")
        if self.scheme == "11stage":
            d = fourth_order_defect(ELEVEN_SIGMA, ELEVEN_ETA, ELEVEN_LAM, ELEVEN_THETA)
            if max(abs(d[0]), abs(d[1])) > 1e-12:
                raise AssertionError("11-stage coefficients violate the fourth-order conditions")

    def micro_steps(self) -> int:
        if self.scheme not in NESTED_SCHEMES:
            return 1
        if self.micro_per_call is not None:
            return self.micro_per_call
        span = 1.0 if self.scheme == "nested-leapfrog" else 0.5
        return max(1, round(span * self.micro_ratio))


@dataclass(frozen=True)
class TrajectoryResult:
    n_steps: int
    inversions: int
    realized_tau: float


# ---------------------------------------------------------------------------
# elementary maps (integrators.py:157-246)
# ---------------------------------------------------------------------------

def _add(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    return kick(a, b, -1.0)      # a - (-1*b) == a + b exactly


def drift(state: MdState, dt: float):
    """q <- wrap(q + dt p) (integrators.py:157-158)."""
    state.q = rotate_links(state.q, state.p, dt)


def kick_gauge(state: MdState, dt: float):
    """p <- p - dt*beta*g, fused force+kick kernel (integrators.py:161-164)."""
    if dt == 0.0:
        return
    state.p = kick_gauge_fused(state.q, state.p, state.beta, dt)


def kick_fermion(state: MdState, dt: float):
    """p <- p - dt*f after the chi/xi solve (integrators.py:172-177)."""
    if dt == 0.0:
        return
    op, chi, xi = state.solve_pair()
    state.p = kick_fermion_fused(op, chi, xi, state.p, dt)


def kick_full(state: MdState, dt: float):
    """p <- p - dt*(F_G + f) (integrators.py:180-186)."""
    if dt == 0.0:
        return
    op, chi, xi = state.solve_pair()
    state.p = kick_fermion_fused(op, chi, xi, state.p, dt, q=state.q, beta=state.beta)


def kick_fg_gauge(state: MdState, b_dt: float, c_dt3: float):
    """Gauge-only force-gradient kick (integrators.py:189-196)."""
    if c_dt3 == 0.0:
        kick_gauge(state, b_dt)
        return
    g = gauge_force(state.q, state.beta)
    fg = fg_gauge_gauge(state.q, state.beta)
    state.p = kick(state.p, g, b_dt, fg, FG_KICK_SIGN * c_dt3)


def _fgh(state, op, chi, xi, weight):
    return fg_fermion_hessian_dot(op, chi, xi, weight, state.tol, counter=state.counter,
                                  exact=state.exact_solves, stop=state.stop, check=False,
                                  infos=state._infos)


def kick_fg_fermion(state: MdState, b_dt: float, c_dt3: float):
    """Fermion kick with the fermion-fermion FG term; 4 inversions (integrators.py:199-209)."""
    if c_dt3 == 0.0:
        kick_fermion(state, b_dt)
        return
    op, chi, xi = state.solve_pair()
    f = fermion_force(op, chi, xi)
    fg = _fgh(state, op, chi, xi, f)
    state.p = kick(state.p, f, b_dt, fg, FG_KICK_SIGN * c_dt3)


def kick_fg_full(state: MdState, b_dt: float, c_dt3: float):
    """Full-action FG kick with all four Hessian pieces; 6 inversions (integrators.py:212-227)."""
    if c_dt3 == 0.0:
        kick_full(state, b_dt)
        return
    op, chi, xi = state.solve_pair()
    f = fermion_force(op, chi, xi)
    g = gauge_force(state.q, state.beta)
    fg = _add(_add(_add(fg_gauge_gauge(state.q, state.beta), gauge_hessian_dot(state.q, state.beta, f)),
                   _fgh(state, op, chi, xi, g)),
              _fgh(state, op, chi, xi, f))
    state.p = kick(state.p, _add(g, f), b_dt, fg, FG_KICK_SIGN * c_dt3)


def kick_fg_approx(state: MdState, b_dt: float, c_dt3: float):
    """Taylor-approximated FG kick: second force at a shifted configuration;
    4 inversions (integrators.py:230-246)."""
    if c_dt3 == 0.0:
        kick_full(state, b_dt)
        return
    op, chi, xi = state.solve_pair()
    force = _add(gauge_force(state.q, state.beta), fermion_force(op, chi, xi))
    q_shift = rotate_links(state.q, force, 2.0 * FG_KICK_SIGN * c_dt3 / b_dt)
    op2 = WilsonDirac(q_shift, state.m0, state.fermion_bc)
    chi2, xi2, rep = chi_xi(op2, state.eta, state.tol, counter=state.counter,
                            exact=state.exact_solves, stop=state.stop, check=False)
    if rep._info is not None:
        state._infos.append(rep._info)
    shifted = _add(gauge_force(q_shift, state.beta), fermion_force(op2, chi2, xi2))
    state.p = kick(state.p, shifted, b_dt)


# ---------------------------------------------------------------------------
# inner (micro) flows of the gauge-only system (integrators.py:253-271)
# ---------------------------------------------------------------------------

def inner_leapfrog(state: MdState, span: float, m: int):
    """M micro leapfrog steps, one resident kernel for the whole flow."""
    q, p = state.q.clone(), state.p.clone()
    g = geom_of(q)
    _lib.ctx().call("sch_inner_leapfrog", _lib.ptr(q), _lib.ptr(p), float(state.beta), float(span),
                    int(m), n_chains(q), g.L, g.T)
    state.q, state.p = q, p


def inner_fg(state: MdState, span: float, m: int, fgc: float):
    """M micro 5-stage force-gradient steps of the gauge action."""
    delta = span / m
    c_d3 = fgc * delta**3
    for _ in range(m):
        kick_gauge(state, delta / 6.0)
        drift(state, 0.5 * delta)
        kick_fg_gauge(state, 2.0 * delta / 3.0, c_d3)
        drift(state, 0.5 * delta)
        kick_gauge(state, delta / 6.0)


# ---------------------------------------------------------------------------
# macro steps as programs.  Entry: (map, weight(h)) where map is one of
#   "D" drift, "K" kick_full, "Kf" kick_fermion, "G<kind>" FG kick with
#   b = weight(h), c = fgc*h^3, "I<kind>" inner flow over span weight(h).
# ---------------------------------------------------------------------------

def _sixth(h):
    return h / 6.0


def _half(h):
    return 0.5 * h


def _two_thirds(h):
    return 2.0 * h / 3.0


def _one(h):
    return h


def _eleven_program():
    s, e, l, t = ELEVEN_SIGMA, ELEVEN_ETA, ELEVEN_LAM, ELEVEN_THETA
    w_half = 0.5 * (1.0 - 2.0 * (l + s))
    c_mid = 1.0 - 2.0 * (t + e)
    prog = []
    for kw, dw in ((s, e), (l, t), (w_half, c_mid), (w_half, t), (l, e), (s, None)):
        prog.append(("K", lambda h, kw=kw: kw * h))
        if dw is not None:
            prog.append(("D", lambda h, dw=dw: dw * h))
    return tuple(prog)


PROGRAMS = {
    "leapfrog": (("K", _half), ("D", _one), ("K", _half)),
    "5stage": (("K", _sixth), ("D", _half), ("K", _two_thirds), ("D", _half), ("K", _sixth)),
    "5stage-fg": (("K", _sixth), ("D", _half), ("Gfull", _two_thirds), ("D", _half), ("K", _sixth)),
    "fg-approx": (("K", _sixth), ("D", _half), ("Gapprox", _two_thirds), ("D", _half), ("K", _sixth)),
    "11stage": _eleven_program(),
    "nested-leapfrog": (("Kf", _half), ("Ileapfrog", _one), ("Kf", _half)),
    "nested-5stage": (("Kf", _sixth), ("Ileapfrog", _half), ("Kf", _two_thirds),
                      ("Ileapfrog", _half), ("Kf", _sixth)),
    "nested-fg": (("Kf", _sixth), ("Ifg", _half), ("Gfermion", _two_thirds), ("Ifg", _half),
                  ("Kf", _sixth)),
    "adapted-nested-fg": (("Kf", _sixth), ("Ileapfrog", _half), ("Gfermion", _two_thirds),
                          ("Ileapfrog", _half), ("Kf", _sixth)),
}

_FG_KICKS = {"Gfull": kick_fg_full, "Gapprox": kick_fg_approx, "Gfermion": kick_fg_fermion}


def _make_step(program):
    def step(state: MdState, h: float, m: int, fgc: float):
        for name, weight in program:
            w = weight(h)
            if name == "D":
                drift(state, w)
            elif name == "K":
                kick_full(state, w)
            elif name == "Kf":
                kick_fermion(state, w)
            elif name in _FG_KICKS:
                _FG_KICKS[name](state, w, fgc * h**3)
            elif name == "Ileapfrog":
                inner_leapfrog(state, w, m)
            elif name == "Ifg":
                inner_fg(state, w, m, fgc)
            else:
                raise KeyError(name)
    return step


SCHEMES = {name: _make_step(prog) for name, prog in PROGRAMS.items()}

step_leapfrog = SCHEMES["leapfrog"]
step_5stage = SCHEMES["5stage"]
step_5stage_fg = SCHEMES["5stage-fg"]
step_fg_approx = SCHEMES["fg-approx"]
step_11stage = SCHEMES["11stage"]
step_nested_leapfrog = SCHEMES["nested-leapfrog"]
step_nested_5stage = SCHEMES["nested-5stage"]
step_nested_fg = SCHEMES["nested-fg"]
step_adapted_nested_fg = SCHEMES["adapted-nested-fg"]


def integrate_trajectory(state: MdState, spec: IntegratorSpec, tau: float,
                         check: bool = True) -> TrajectoryResult:
    """round(tau/h) macro steps in place; returns the step count, the
    inversions spent (reference convention) and n_steps*h (integrators.py:365-382).
    ``check=False`` leaves the SolverError check of the trajectory's solves to
    the caller (``state.check_solves()``), so nothing synchronises with the host."""
    if not tau > 0:
        raise ValueError(f"trajectory length must be positive, got {tau}")
    n_steps = max(1, round(tau / spec.h))
    step = SCHEMES[spec.scheme]
    m = spec.micro_steps()
    before = state.counter.count
    for _ in range(n_steps):
        step(state, spec.h, m, spec.fg_coefficient)
    if check:
        state.check_solves()
    return TrajectoryResult(n_steps=n_steps, inversions=state.counter.count - before,
                            realized_tau=n_steps * spec.h)
