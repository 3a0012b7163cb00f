"""Independent-chain ensembles across GPUs (BASELINE configs 3-4).

One process per GPU.  Chains are partitioned into contiguous ranges, one per
rank; every chain keeps its own RNG stream (chain c <-> ``make_rng(seed,
stream=c)`` in parity mode, Philox key (seed, c) in bench mode), so results
do not depend on the number of ranks.  There is no communication while
trajectories run; the only collective is the final all-gather of per-chain
observables (dH, accept, plaquette), which goes over NCCL on GPUs and gloo
in the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class ChainShard:
    """Contiguous chain range [start, start + count) owned by one rank."""

    rank: int
    world: int
    start: int
    count: int
    total: int

    @property
    def stop(self) -> int:
        return self.start + self.count


def shard_chains(total: int, world: int, rank: int) -> ChainShard:
    """Balanced contiguous partition: the first ``total % world`` ranks get one
    extra chain."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if total < 0:
        raise ValueError("negative chain count")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return ChainShard(rank, world, start, base + (1 if rank < extra else 0), total)


def chain_rngs(seed: int, shard: ChainShard):
    """Parity-mode generators of the shard's chains (global stream ids)."""
    from .lattice import make_rng
    return [make_rng(seed, stream=c) for c in range(shard.start, shard.stop)]


def gather_observables(local: dict, shard: ChainShard, group=None, device=None) -> dict:
    """All-gather per-chain float64 observables into global chain order.

    ``local`` maps names to 1-D arrays of length ``shard.count``.  With a
    single rank (or no initialised process group) the input is returned as
    numpy arrays."""
    names = sorted(local)
    if shard.world == 1 or not dist.is_initialized():
        return {k: np.asarray(local[k], dtype=np.float64) for k in names}
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(group) == "nccl" else torch.device("cpu")
    counts = [shard_chains(shard.total, shard.world, r).count for r in range(shard.world)]
    width = max(counts)
    block = torch.zeros((len(names), width), dtype=torch.float64, device=device)
    for i, k in enumerate(names):
        v = torch.as_tensor(np.asarray(local[k], dtype=np.float64))
        block[i, :v.numel()] = v.to(device)
    parts = [torch.empty_like(block) for _ in range(shard.world)]
    dist.all_gather(parts, block, group=group)
    out = {}
    for i, k in enumerate(names):
        out[k] = np.concatenate([parts[r][i, :counts[r]].cpu().numpy() for r in range(shard.world)])
    return out


def summarize(obs: dict) -> dict:
    """Ensemble averages of a gathered observable set."""
    dh = obs.get("dh")
    out = {}
    if dh is not None:
        out["mean_abs_dh"] = float(np.mean(np.abs(dh)))
        out["exp_minus_dh"] = float(np.mean(np.exp(-dh)))
    if "accepted" in obs:
        out["acceptance"] = float(np.mean(obs["accepted"]))
    if "plaquette" in obs:
        out["plaquette"] = float(np.mean(obs["plaquette"]))
    return out
