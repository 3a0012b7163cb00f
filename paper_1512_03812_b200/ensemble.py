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


# ---------------------------------------------------------------------------
# checkpoint / resume
# ---------------------------------------------------------------------------

def save_checkpoint(path, q, rng, shard: ChainShard | None = None, trajectory: int = 0,
                    meta: dict | None = None) -> None:
    """Write a shard's links and its chains' RNG positions to one .npz.

    ``rng`` is a ``NumpyDeviceRng`` (device streams) or a list of host
    Generators (parity mode); either way the file stores NumPy Philox states,
    so a run can resume on the GPU or be handed to the reference's own
    ``hmc_update`` per chain.  Links are the reference layout (B, 2, L, T)."""
    from .lattice import NumpyDeviceRng, to_numpy
    qn = to_numpy(q)
    states = rng.get_states() if isinstance(rng, NumpyDeviceRng) else [g.bit_generator.state for g in rng]
    if len(states) != qn.shape[0]:
        raise ValueError(f"{len(states)} RNG streams for {qn.shape[0]} chains")
    shard = shard or ChainShard(0, 1, 0, qn.shape[0], qn.shape[0])
    np.savez(path, format=np.array("schwinger-b200-ensemble v1"), q=qn,
             ctr=np.stack([s["state"]["counter"] for s in states]).astype(np.uint64),
             key=np.stack([s["state"]["key"] for s in states]).astype(np.uint64),
             buf=np.stack([s["buffer"] for s in states]).astype(np.uint64),
             pos=np.array([s["buffer_pos"] for s in states], dtype=np.int32),
             shard=np.array([shard.rank, shard.world, shard.start, shard.count, shard.total]),
             trajectory=np.int64(trajectory), meta=np.array(repr(meta or {})))


def load_checkpoint(path, device_rng: bool = True):
    """Inverse of ``save_checkpoint``: (q on the GPU, rng, shard, trajectory).

    ``device_rng`` selects a ``NumpyDeviceRng`` continuing every stream on the
    GPU; otherwise host Generators are returned."""
    import ast
    from .lattice import NumpyDeviceRng, as_links
    z = np.load(path)
    if str(z["format"]) != "schwinger-b200-ensemble v1":
        raise ValueError(f"{path}: not an ensemble checkpoint")
    states = [{"bit_generator": "Philox", "state": {"counter": z["ctr"][c], "key": z["key"][c]},
               "buffer": z["buf"][c], "buffer_pos": int(z["pos"][c]), "has_uint32": 0,
               "uinteger": 0} for c in range(z["ctr"].shape[0])]
    if device_rng:
        rng = NumpyDeviceRng(0, len(states))
        rng.set_states(states)
    else:
        rng = []
        for s in states:
            g = np.random.Generator(np.random.Philox(key=[0, 0]))
            g.bit_generator.state = s
            rng.append(g)
    r, w, start, count, total = (int(v) for v in z["shard"])
    meta = ast.literal_eval(str(z["meta"]))
    return as_links(z["q"]), rng, ChainShard(r, w, start, count, total), int(z["trajectory"]), meta
