"""HMC update cycle on the B200: heatbaths, trajectory, Hamiltonian,
Metropolis; the batched fixed-start |dH| measurement; thermalization; and the
independent-chain ensemble update used by the benchmark.

Mirror of ``schwinger.hmc`` (pkg/src/schwinger/hmc.py).  ``hmc_update`` and
``measure_dh`` keep the reference signatures, draw order and return types
(dH as a Python float, reject returns the caller's original object).
``hmc_update_ensemble`` is the B200 addition: B chains advanced together with
per-chain CG stopping, per-chain RNG streams and per-chain Metropolis — the
same result as B independent ``hmc_update`` calls.
"""

from __future__ import annotations

import logging
import time
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _lib
from .config import HmcConfig
from .fermion import InversionCounter, WilsonDirac, draw_phi, pseudofermion_heatbath, spinor_dot
from .gauge import avg_plaquette, gauge_action
from .fermion import SolverError
from .integrators import (FG_KICK_SIGN, INVERSIONS_PER_STEP, IntegratorSpec, MdState, TrajectoryResult,
                          integrate_trajectory)
from .lattice import (DeviceRng, LatticeGeom, NumpyDeviceRng, as_links, as_spinor, cold_start,
                      kick, kinetic_energy,
                      sample_momenta)

log = logging.getLogger("schwinger")


@dataclass(frozen=True)
class TrajectoryStats:
    dh: float
    accepted: bool
    inversions: int
    n_steps: int
    wall_time: float


@dataclass(frozen=True)
class DhMeasurement:
    """|dH| statistics over independent trajectories from one configuration."""

    dh: np.ndarray
    mean_abs: float
    stderr: float
    acceptance: float
    inversions_per_traj: int
    n_steps: int
    wall_per_traj: float


@dataclass(frozen=True)
class EnsembleStats:
    """Per-chain outcome of one ensemble trajectory."""

    dh: np.ndarray
    accepted: np.ndarray
    inversions: int          # per chain, reference convention
    n_steps: int
    wall_time: float


def hamiltonian(state: MdState) -> torch.Tensor:
    """H = (1/2) sum p^2 + S_G + S_F per chain; one normal solve, shared with
    an adjacent kick at the same links when ``reuse_solves`` (hmc.py:44-51)."""
    kin = kinetic_energy(state.p)
    s_g = gauge_action(state.q, state.beta)
    _, _, xi = state.solve_pair()
    s_f = spinor_dot(state.eta, xi).real.contiguous()
    return kick(kick(kin, s_g, -1.0), s_f, -1.0)   # (kin + s_g) + s_f, on our kernel


def metropolis(dh: float, rng) -> bool:
    """Accept with probability min(1, exp(-dH)); draws only when dH > 0 (hmc.py:54-60)."""
    if not np.isfinite(dh):
        raise ValueError(f"non-finite energy change {dh}")
    if dh <= 0.0:
        return True
    return bool(rng.random() < np.exp(-dh))


def _spec_of(config: HmcConfig) -> IntegratorSpec:
    return IntegratorSpec(scheme=config.scheme, h=config.h, micro_per_call=config.micro_per_call,
                          micro_ratio=config.micro_ratio)


def _sync():
    torch.cuda.synchronize()


def hmc_update(q, config: HmcConfig, rng, counter: InversionCounter | None = None,
               reuse_solves: bool = True):
    """One HMC update (hmc.py:69-95); returns (links, TrajectoryStats).

    On rejection the caller's object is handed back untouched."""
    counter = counter if counter is not None else InversionCounter()
    geom = LatticeGeom(config.L, config.T)
    q_dev = as_links(q)
    p = sample_momenta(rng, geom)
    if config.quenched:
        eta = torch.zeros(geom.spinor_shape(), dtype=torch.complex128, device=q_dev.device)
    else:
        eta = pseudofermion_heatbath(WilsonDirac(q_dev, config.m0, config.fermion_bc), rng)
    state = MdState(q=q_dev.clone(), p=p, eta=eta, beta=config.beta, m0=config.m0,
                    tol=config.cg_tol, counter=counter, fermion_bc=config.fermion_bc,
                    stop="per_chain", reuse_solves=reuse_solves)
    h_start = hamiltonian(state)
    _sync()
    t0 = time.perf_counter()
    result = integrate_trajectory(state, _spec_of(config), config.tau)
    _sync()
    wall = time.perf_counter() - t0
    h_end = hamiltonian(state)
    state.check_solves()
    dh = float(kick(h_end, h_start, 1.0).item())
    accepted = metropolis(dh, rng)
    stats = TrajectoryStats(dh=dh, accepted=accepted, inversions=result.inversions,
                            n_steps=result.n_steps, wall_time=wall)
    return (state.q if accepted else q), stats


def measure_dh(q0, config: HmcConfig, rng, n_samples: int | None = None,
               reuse_solves: bool = True) -> DhMeasurement:
    """Mean |dH| over n independent momentum/pseudofermion draws from one
    configuration, evolved as one batch with global CG stopping; no
    Metropolis step (hmc.py:98-130)."""
    n = n_samples if n_samples is not None else config.n_samples
    geom = LatticeGeom(config.L, config.T)
    counter = InversionCounter()
    q0 = as_links(q0)
    p = sample_momenta(rng, geom, batch=n)
    if config.quenched:
        eta = torch.zeros(geom.spinor_shape(n), dtype=torch.complex128, device=q0.device)
    else:
        eta = pseudofermion_heatbath(WilsonDirac(q0, config.m0, config.fermion_bc), rng, batch=n)
    q = q0.expand((n,) + tuple(q0.shape)).contiguous()
    state = MdState(q=q, p=p, eta=eta, beta=config.beta, m0=config.m0, tol=config.cg_tol,
                    counter=counter, fermion_bc=config.fermion_bc, stop="batch_global",
                    reuse_solves=reuse_solves)
    h_start = hamiltonian(state)
    _sync()
    t0 = time.perf_counter()
    result = integrate_trajectory(state, _spec_of(config), config.tau)
    _sync()
    wall = time.perf_counter() - t0
    h_end = hamiltonian(state)
    state.check_solves()
    dh = kick(h_end, h_start, 1.0).cpu().numpy().astype(np.float64)
    ad = np.abs(dh)
    mean_abs = float(np.mean(ad))
    stderr = float(np.std(ad, ddof=1) / np.sqrt(n)) if n > 1 else 0.0
    acceptance = float(np.mean(np.minimum(1.0, np.exp(-dh))))
    return DhMeasurement(dh=dh, mean_abs=mean_abs, stderr=stderr, acceptance=acceptance,
                         inversions_per_traj=result.inversions, n_steps=result.n_steps,
                         wall_per_traj=wall / n)


def thermalize(config: HmcConfig, rng, on_solver_error: str = "raise"):
    """Cold start + n_thermalize leapfrog updates with step annealing
    (hmc.py:133-155).  Returns (links on the device, plaquette history).

    ``on_solver_error="reject"`` (not a reference option) counts an update
    whose CG hit the cap as rejected instead of raising.  At the paper's
    point (m0 = -0.231367, beta = 1) the first cold-start trajectories are
    unstable (|dH| ~ 1e7 in the reference run too), so rounding-level
    differences grow until a near-singular D appears on one side and not the
    other; burn-in only, the chain after it is an ordinary HMC chain."""
    if on_solver_error not in ("raise", "reject"):
        raise ValueError(f"on_solver_error must be 'raise' or 'reject', got {on_solver_error!r}")
    geom = LatticeGeom(config.L, config.T)
    q = cold_start(geom)
    tc = replace(config, scheme="leapfrog", h=min(config.h, 0.1), micro_per_call=None)
    block, hits, history = 20, 0, []
    for i in range(config.n_thermalize):
        try:
            q, stats = hmc_update(q, tc, rng)
        except SolverError as exc:
            if on_solver_error == "raise":
                raise
            log.warning("thermalize: update %d rejected: %s", i, exc)
            history.append(history[-1] if history else float(avg_plaquette(q).item()))
            if (i + 1) % block == 0:
                if hits < 0.8 * block:
                    tc = replace(tc, h=tc.h * 0.7)
                    log.info("thermalize: lowering step size to %.4g", tc.h)
                hits = 0
            continue
        hits += stats.accepted
        history.append(float(avg_plaquette(q).item()))
        if (i + 1) % block == 0:
            if hits < 0.8 * block:
                tc = replace(tc, h=tc.h * 0.7)
                log.info("thermalize: lowering step size to %.4g", tc.h)
            hits = 0
    return q, history


# ---------------------------------------------------------------------------
# chain ensemble (BASELINE configs 3-4)
# ---------------------------------------------------------------------------

def hmc_update_ensemble(q, config: HmcConfig, rngs=None, device_rng: DeviceRng | None = None,
                        counter: InversionCounter | None = None, reuse_solves: bool = True):
    """Advance B independent chains by one HMC update each.

    ``q`` is (B, 2, L, T).  Parity mode: ``rngs`` is a list of B NumPy
    generators (chain c == ``make_rng(seed, stream=c)``) and every chain sees
    exactly the draws an unbatched ``hmc_update`` would make.  Bench mode:
    ``device_rng`` draws momenta, pseudofermions and Metropolis uniforms on
    the GPU.  Returns (links, EnsembleStats)."""
    if (rngs is None) == (device_rng is None):
        raise ValueError("pass exactly one of rngs (parity mode) or device_rng (bench mode)")
    if device_rng is not None:
        out, pending = hmc_update_ensemble_async(q, config, device_rng, counter, reuse_solves)
        return out, pending.resolve()
    return _ensemble_update(q, config, rngs, None, counter, reuse_solves, sync=True)


class PendingEnsembleStats:
    """Outcome of an ensemble update issued without any host synchronisation:
    per-chain dH and accept flags still on the device.  ``resolve()`` reads
    them back, raises SolverError / ValueError exactly as the synchronous
    call would, and returns the EnsembleStats."""

    def __init__(self, state, result, dh_dev, acc_dev, t0):
        self._state, self._result = state, result
        self.dh_dev, self.acc_dev = dh_dev, acc_dev
        self._t0 = t0
        self._stream = torch.cuda.current_stream(dh_dev.device)
        self._stats = None

    def resolve(self) -> "EnsembleStats":
        if self._stats is None:
            with torch.cuda.stream(self._stream):   # read back in the issuing stream's order
                self._state.check_solves()
                dh = self.dh_dev.cpu().numpy()
                acc_h = self.acc_dev.cpu().numpy()
            if (acc_h < 0).any():
                raise ValueError(f"non-finite energy change {dh[acc_h < 0][0]}")
            self._stats = EnsembleStats(dh=dh, accepted=acc_h == 1,
                                        inversions=self._result.inversions,
                                        n_steps=self._result.n_steps,
                                        wall_time=time.perf_counter() - self._t0)
        return self._stats


def hmc_update_ensemble_async(q, config: HmcConfig, device_rng, counter=None,
                              reuse_solves: bool = True):
    """Bench-mode ensemble update, issued on torch's current stream with no
    host round trip: returns (links, PendingEnsembleStats).  Sub-ensembles
    issued on different streams run concurrently (each stream has its own
    library context), which fills the GPU during one another's CG tails and
    small kernels.  Rejected / non-finite chains keep their input links."""
    return _ensemble_update(q, config, None, device_rng, counter, reuse_solves, sync=False)


# The trajectory megakernel (csrc/mega.cu): one launch runs H(start), the
# whole adapted-nested-fg trajectory and H(end) of every 16x16 chain, with
# the same arithmetic as the kernel-per-map path below (tests/test_gpu_mega.py).
# Opt-in (SCH_MEGA=1): on cfg3 it measured 161k vs 172k chain-traj/s for the
# kernel-per-map path — the solver inlined into the larger kernel issues at
# 62 % FP64-pipe activity instead of 70 %.
USE_MEGA = __import__("os").environ.get("SCH_MEGA", "0") == "1"


def _mega_eligible(config: HmcConfig, reuse_solves: bool) -> bool:
    return (USE_MEGA and reuse_solves and config.scheme == "adapted-nested-fg"
            and config.L == 16 and config.T == 16 and config.fermion_bc == "periodic"
            and not config.quenched)


class _MegaStatus:
    """Per-chain CG failure flags of a megakernel trajectory (the CgInfo
    interface the update paths check)."""

    def __init__(self, status, maxiter):
        self.status_dev, self._maxiter = status, maxiter

    def raise_if_failed(self):
        if bool(self.status_dev.ne(0).any().item()):
            raise SolverError(f"CG exceeded {self._maxiter} iterations", float("nan"))


class _MegaState:
    """What PendingEnsembleStats / EnsembleUpdateGraph need from an MdState:
    the final links and the solver checks."""

    def __init__(self, q, status, maxiter):
        self.q = q
        self._infos = [_MegaStatus(status, maxiter)]

    def check_solves(self):
        for i in self._infos:
            i.raise_if_failed()


def _mega_trajectory(q, p, eta, config: HmcConfig, counter):
    """(q_end, dH, state, TrajectoryResult) of one adapted-nested-fg trajectory
    per chain in one kernel (same scalars as integrators.PROGRAMS)."""
    from .fermion import DEFAULT_MAXITER
    spec = _spec_of(config)
    h = spec.h
    n = max(1, round(config.tau / h))
    B = q.shape[0]
    q_end = torch.empty_like(q)
    dh = torch.empty((B,), dtype=torch.float64, device=q.device)
    status = torch.empty((B,), dtype=torch.int32, device=q.device)
    iters = torch.empty((B,), dtype=torch.int32, device=q.device)
    from . import fermion as _F
    prof = _F.CG_PROFILE   # bench instrumentation: the megakernel is the step's CG time
    if prof is not None:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
    _lib.ctx().call("sch_traj_anfg16", _lib.ptr(q), _lib.ptr(p), _lib.ptr(eta), _lib.ptr(q_end),
                    _lib.ptr(dh), _lib.ptr(status), _lib.ptr(iters), B, float(config.beta),
                    float(config.m0), float(config.cg_tol), int(DEFAULT_MAXITER), h / 6.0,
                    2.0 * h / 3.0, FG_KICK_SIGN * (spec.fg_coefficient * h**3), 0.5 * h, int(n),
                    int(spec.micro_steps()))
    if prof is not None:
        ev1.record()
        prof.append((ev0, ev1, iters, config.L * config.T))
    inv = INVERSIONS_PER_STEP[config.scheme] * n
    counter.add(inv + 4)   # + the two Hamiltonian solves, as the kernel-per-map path counts
    return q_end, dh, _MegaState(q_end, status, DEFAULT_MAXITER), TrajectoryResult(
        n_steps=n, inversions=inv, realized_tau=n * h)


def _ensemble_update(q, config, rngs, device_rng, counter, reuse_solves, sync):
    q = as_links(q)
    if q.ndim != 4:
        raise ValueError("hmc_update_ensemble expects links of shape (B, 2, L, T)")
    B = q.shape[0]
    geom = LatticeGeom(config.L, config.T)
    counter = counter if counter is not None else InversionCounter()
    if rngs is not None:
        if len(rngs) != B:
            raise ValueError(f"need one generator per chain ({B}), got {len(rngs)}")
        ps, phis = [], []
        for r in rngs:
            ps.append(r.standard_normal(geom.links_shape()))
            if not config.quenched:
                phis.append(draw_phi(r, config.L, config.T))
        p = as_links(np.stack(ps))
        phi = as_spinor(np.stack(phis)) if phis else None
    elif isinstance(device_rng, NumpyDeviceRng):   # the reference's streams, drawn on device
        if device_rng.n != B:
            raise ValueError(f"device streams for {device_rng.n} chains, links for {B}")
        p, phi = device_rng.heatbath(geom, config.quenched)
    else:
        p = device_rng.normal(B, geom.links_shape())
        phi = None if config.quenched else device_rng.complex_normal(B, geom.spinor_shape(),
                                                                     1.0 / np.sqrt(2.0))
    if config.quenched:
        eta = torch.zeros(geom.spinor_shape(B), dtype=torch.complex128, device=q.device)
    else:
        eta = WilsonDirac(q, config.m0, config.fermion_bc).apply_dag(phi)
    t0 = time.perf_counter()
    if _mega_eligible(config, reuse_solves):
        q_end, dh_dev, state, result = _mega_trajectory(q, p, eta, config, counter)
        if sync:
            state.check_solves()
    else:
        state = MdState(q=q.clone(), p=p, eta=eta, beta=config.beta, m0=config.m0,
                        tol=config.cg_tol, counter=counter, fermion_bc=config.fermion_bc,
                        stop="per_chain", reuse_solves=reuse_solves)
        h_start = hamiltonian(state)
        result = integrate_trajectory(state, _spec_of(config), config.tau, check=sync)
        h_end = hamiltonian(state)
        dh_dev = kick(h_end, h_start, 1.0)
    if device_rng is not None:
        if isinstance(device_rng, NumpyDeviceRng):
            acc = device_rng.metropolis(dh_dev)
        else:
            u = device_rng.uniform(B)
            acc = torch.empty((B,), dtype=torch.int32, device=q.device)
            _lib.ctx().call("sch_metropolis", _lib.ptr(dh_dev), _lib.ptr(u), _lib.ptr(acc), B)
        out = torch.empty_like(q)
        _lib.ctx().call("sch_select_chains", _lib.ptr(acc), _lib.ptr(state.q), _lib.ptr(q),
                        _lib.ptr(out), B, q[0].numel())
        pending = PendingEnsembleStats(state, result, dh_dev, acc, t0)
        return (out, pending.resolve()) if sync else (out, pending)
    state.check_solves()
    dh = dh_dev.cpu().numpy()
    accepted = np.array([metropolis(float(d), r) for d, r in zip(dh, rngs)], dtype=bool)
    acc = torch.from_numpy(accepted.astype(np.int32)).to(q.device)
    out = torch.empty_like(q)
    _lib.ctx().call("sch_select_chains", _lib.ptr(acc), _lib.ptr(state.q), _lib.ptr(q),
                    _lib.ptr(out), B, q[0].numel())
    wall = time.perf_counter() - t0
    return out, EnsembleStats(dh=dh, accepted=accepted, inversions=result.inversions,
                              n_steps=result.n_steps, wall_time=wall)


class EnsembleUpdateGraph:
    """One ensemble HMC update captured once as a CUDA graph and replayed
    (whole-trajectory on-device execution).

    ``step()`` replays heatbaths, both Hamiltonians, the whole trajectory,
    Metropolis and the accept/reject select with one graph launch: no Python,
    no per-kernel launch cost, the chains' state (links, the NumPy-stream
    RNG) advancing in place on the device.  Values are identical to
    ``hmc_update_ensemble`` with the same ``NumpyDeviceRng``.  Requires the
    resident or cluster-resident CG engines (V <= 1024, or 64^2): the
    streaming engine runs its own device-side graph."""

    def __init__(self, q, config: HmcConfig, device_rng: NumpyDeviceRng, reuse_solves: bool = True,
                 cg_profile: list | None = None):
        if not isinstance(device_rng, NumpyDeviceRng):
            raise TypeError("graph capture needs the device-resident NumpyDeviceRng streams")
        V = config.L * config.T
        if not (V <= 1024 or (config.L == 64 and config.T == 64)):
            raise ValueError("graph capture needs a resident CG engine (V <= 1024 or 64x64)")
        self.q = as_links(q).clone()
        self.rng = device_rng
        self.config = config
        self._stream = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        self._stream.wait_stream(main)
        saved = device_rng.state.clone()
        with torch.cuda.stream(self._stream):   # warm-up: library context, workspace, attributes
            hmc_update_ensemble_async(self.q, config, device_rng, InversionCounter(), reuse_solves)
        self._stream.synchronize()
        device_rng.state.copy_(saved)            # the warm-up's draws are given back
        self.graph = torch.cuda.CUDAGraph()
        counter = InversionCounter()
        # cg_profile: the CG launches' events and iteration tensors of the
        # captured update (external event nodes: each replay refreshes them)
        from . import fermion as _fermion
        saved_prof, _fermion.CG_PROFILE = _fermion.CG_PROFILE, cg_profile
        launches0 = _lib.launch_count()
        try:
            with torch.cuda.graph(self.graph, stream=self._stream):
                out, pend = hmc_update_ensemble_async(self.q, config, device_rng, counter,
                                                      reuse_solves)
                self.q.copy_(out)
                # any CG of this replay at its cap (0/1), formed inside the graph
                flags = [i.status_dev.reshape(-1) for i in pend._state._infos]
                self.failed = (torch.cat(flags).amax() if flags
                               else torch.zeros((), dtype=torch.int32, device=self.q.device))
        finally:
            _fermion.CG_PROFILE = saved_prof
        self.launches_per_replay = _lib.launch_count() - launches0   # our kernels in the graph
        self._pending = pend
        self._infos = list(pend._state._infos)
        self.inversions = pend._result.inversions
        self.n_steps = pend._result.n_steps
        main.wait_stream(self._stream)

    def step(self):
        """Replay one update on the current stream; returns the pending
        per-chain (dH, accept) tensors (read them with ``stats()``;
        ``self.failed`` is 1 when a CG solve of the replay hit its cap)."""
        self.graph.replay()
        return self._pending.dh_dev, self._pending.acc_dev

    def stats(self) -> "EnsembleStats":
        """Host read-back of the last replay (raises like hmc_update_ensemble)."""
        if self._infos:
            bad = torch.cat([i.status_dev.reshape(-1) for i in self._infos]).ne(0).any()
            if bool(bad.item()):
                for i in self._infos:
                    i.raise_if_failed()
        dh = self._pending.dh_dev.cpu().numpy()
        acc = self._pending.acc_dev.cpu().numpy()
        if (acc < 0).any():
            raise ValueError(f"non-finite energy change {dh[acc < 0][0]}")
        return EnsembleStats(dh=dh, accepted=acc == 1, inversions=self.inversions,
                             n_steps=self.n_steps, wall_time=float("nan"))
