"""Test infrastructure: the oracle spread over the host cores.

Element-wise parity at BASELINE.json's full sizes (tests/test_gpu_fullsize.py)
needs the oracle on thousands of chains.  Every chain of these workloads is an
independent problem, so the batch is cut into contiguous chunks and each
chunk runs the oracle's own batched code (per-chain CG stop, or one
unbatched `hmc_update` per chain) in a separate process.  Nothing here is a
product path: only tests/ and bench.py's CPU legs import it.
"""

from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _pool(n):
    # spawn: the caller may hold a CUDA context; the workers only run NumPy
    return mp.get_context("spawn").Pool(n, initializer=_init)


def _init():
    os.environ["OMP_NUM_THREADS"] = "1"


def _cg_chunk(args):
    from oracle import schwinger_oracle as O
    q, b, m0, tol, bc = args
    x, it, _ = O.cg_normal(O.fermion_links(q, bc), m0, b, tol, stop="per_chain")
    return x, it


def cg_per_chain(q, b, m0, tol, bc="periodic", procs=None):
    """Oracle per-chain CG (cg_normal stop='per_chain', the semantics of one
    unbatched reference call per chain, fermion.py:171-217) for every chain of
    the batch: returns (x (B,L,T,2), iterations (B,))."""
    procs = procs or cores()
    B = q.shape[0]
    n = max(1, min(B, 4 * procs))
    edges = np.linspace(0, B, n + 1).astype(int)
    work = [(q[a:e], b[a:e], m0, tol, bc) for a, e in zip(edges[:-1], edges[1:]) if e > a]
    with _pool(procs) as pool:
        res = pool.map(_cg_chunk, work)
    return np.concatenate([r[0] for r in res]), np.concatenate([r[1] for r in res])


def _hmc_chunk(args):
    from oracle import schwinger_oracle as O
    chains, seed, cfg_kw, n_traj = args
    cfg = O.Config(**cfg_kw)
    out = []
    for c in chains:
        rng = O.make_rng(seed, int(c))
        q = O.hot_start(rng, cfg.L, cfg.T)
        q0 = q
        dh, acc, inv = [], [], []
        for _ in range(n_traj):
            q, s = O.hmc_update(q, cfg, rng)
            dh.append(s["dh"])
            acc.append(s["accepted"])
            inv.append(s["inversions"])
        out.append((int(c), q0, q, np.array(dh), np.array(acc), np.array(inv)))
    return out


def hmc_chains(chains, seed, cfg_kw, n_traj=1, procs=None):
    """Independent oracle chains: chain c = hot_start(make_rng(seed, c)) then
    `n_traj` hmc_update calls on the same generator (hmc.py:69-95).  Returns
    {c: (q_start, q_end, dh[n_traj], accepted[n_traj], inversions[n_traj])}."""
    procs = procs or cores()
    chains = list(chains)
    n = max(1, min(len(chains), 4 * procs))
    parts = [chains[i::n] for i in range(n)]
    with _pool(procs) as pool:
        res = pool.map(_hmc_chunk, [(p, seed, cfg_kw, n_traj) for p in parts if p])
    return {c: rest for chunk in res for (c, *rest) in chunk}
