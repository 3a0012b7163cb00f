"""Pure-gauge sector on the B200: plaquettes, Wilson action, force and the
gauge force-gradient pieces.  Mirror of ``schwinger.gauge``
(pkg/src/schwinger/gauge.py); each function launches the sm_100a kernel
named in its docstring."""

from __future__ import annotations

import torch

from . import _lib
from .lattice import as_links, geom_of, n_chains, squeeze_chain


def _geo(q):
    g = geom_of(q)
    return n_chains(q), g.L, g.T


def plaq_angles(q) -> torch.Tensor:
    """q0(n) + q1(n+x) - q0(n+t) - q1(n) per site (gauge.py:21-24); kernel k_plaq_angles."""
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty(q.shape[:-3] + (L, T), dtype=torch.float64, device=q.device)
    _lib.ctx().call("sch_plaquette_angles", _lib.ptr(q), _lib.ptr(out), B, L, T)
    return out


def _plaquette_stencil(q, K: int) -> torch.Tensor:
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty(((K,) if K > 1 else ()) + tuple(q.shape), dtype=torch.complex128,
                      device=q.device)
    _lib.ctx().call("sch_plaquette_stencil", _lib.ptr(q), _lib.ptr(out), K, B, L, T)
    return out


def oriented_plaquettes(q) -> torch.Tensor:
    """P1(n, mu): the plaquette traversed starting along mu — e^{i theta} for
    mu=0, its conjugate for mu=1 — shape (..., 2, L, T) (gauge.py:62-67)."""
    return _plaquette_stencil(q, 1)


def plaquette_stencil(q) -> torch.Tensor:
    """The eight translates P1..P8 of the mu-oriented plaquette attached to
    link (n, mu), shape (8, ..., 2, L, T) (gauge.py:70-95):
    P2 = P1(n-nu), P3 = P1(n+mu), P4 = P1(n+nu), P5 = P1(n-mu),
    P6 = P1(n-mu-nu), P7 = P1(n-2nu), P8 = P1(n-nu+mu)."""
    return _plaquette_stencil(q, 8)


def plaquettes(q) -> torch.Tensor:
    """exp(i * plaquette angle) (gauge.py:27-29), via the sincos link-cache kernel."""
    th = plaq_angles(q)
    B = n_chains(th, 2)
    L, T = th.shape[-2:]
    # sch_links_to_u maps a [B][2][L][T] angle field; feed the plaquettes as
    # the first "direction" of a padded field.
    pad = torch.zeros((B, 2, L, T), dtype=torch.float64, device=th.device)
    pad[:, 0] = th.reshape(B, L, T)
    u = torch.empty((B, 2, L, T), dtype=torch.complex128, device=th.device)
    _lib.ctx().call("sch_links_to_u", _lib.ptr(pad), _lib.ptr(u), B, int(L), int(T), 0)
    return u[:, 0].reshape(th.shape).contiguous()


def avg_plaquette(q) -> torch.Tensor:
    """mean cos(theta) per chain (gauge.py:32-34)."""
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty((B,), dtype=torch.float64, device=q.device)
    _lib.ctx().call("sch_avg_plaquette", _lib.ptr(q), _lib.ptr(out), B, L, T)
    return squeeze_chain(out, q)


def gauge_action(q, beta: float) -> torch.Tensor:
    """beta * sum(1 - cos theta) per chain (gauge.py:37-40)."""
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty((B,), dtype=torch.float64, device=q.device)
    _lib.ctx().call("sch_gauge_action", _lib.ptr(q), float(beta), _lib.ptr(out), B, L, T)
    return squeeze_chain(out, q)


def gauge_force(q, beta: float) -> torch.Tensor:
    """beta * g(n, mu) = dS_G/dq (gauge.py:43-59)."""
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty_like(q)
    _lib.ctx().call("sch_gauge_force", _lib.ptr(q), float(beta), _lib.ptr(out), B, L, T)
    return out


def gauge_force_raw(q) -> torch.Tensor:
    """g without the beta factor (gauge.py:43-54)."""
    return gauge_force(q, 1.0)


def kick_gauge_fused(q: torch.Tensor, p: torch.Tensor, beta: float, dt: float) -> torch.Tensor:
    """p - dt * gauge_force(q, beta) in one pass (integrators.py:161-164)."""
    B, L, T = _geo(q)
    out = torch.empty_like(p)
    _lib.ctx().call("sch_kick_gauge", _lib.ptr(q), _lib.ptr(p), float(beta), float(dt),
                    _lib.ptr(out), B, L, T)
    return out


def fg_gauge_gauge(q, beta: float) -> torch.Tensor:
    """Gauge-gauge force-gradient piece C_GG, closed plaquette form (gauge.py:97-107)."""
    q = as_links(q)
    B, L, T = _geo(q)
    out = torch.empty_like(q)
    _lib.ctx().call("sch_fg_gauge_gauge", _lib.ptr(q), float(beta), _lib.ptr(out), B, L, T)
    return out


def gauge_hessian_dot(q, beta: float, w) -> torch.Tensor:
    """2 * sum w * Hess(S_G) for a link field w (gauge.py:110-136)."""
    q, w = as_links(q), as_links(w)
    if q.shape[-3:] != w.shape[-3:]:
        raise ValueError(f"shape mismatch: links {tuple(q.shape)} vs weight {tuple(w.shape)}")
    if q.shape != w.shape:
        shape = torch.broadcast_shapes(q.shape, w.shape)
        q, w = q.expand(shape).contiguous(), w.expand(shape).contiguous()
    B, L, T = _geo(q)
    out = torch.empty_like(q)
    _lib.ctx().call("sch_gauge_hessian_dot", _lib.ptr(q), float(beta), _lib.ptr(w), _lib.ptr(out),
                    B, L, T)
    return out


def fg_fermion_gauge(q, beta: float, fermion_force) -> torch.Tensor:
    """Gauge Hessian contracted with the fermion force (gauge.py:139-142)."""
    return gauge_hessian_dot(q, beta, fermion_force)
