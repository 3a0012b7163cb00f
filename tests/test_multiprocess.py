"""The N>1 host path of the chain ensemble, run as world_size-2 gloo process
groups on the CPU: chain sharding, per-chain stream assignment, and the final
all-gather of per-chain observables (the only collective of configs 3-4)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1512_03812_b200.ensemble import chain_rngs, gather_observables, shard_chains, summarize


def test_shard_chains_partition_is_balanced_and_complete():
    for total in (0, 1, 7, 8, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            shards = [shard_chains(total, world, r) for r in range(world)]
            assert shards[0].start == 0 and shards[-1].stop == total
            for a, b in zip(shards, shards[1:]):
                assert a.stop == b.start
            counts = [s.count for s in shards]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        shard_chains(8, 2, 2)


def test_chain_streams_do_not_depend_on_world_size():
    """Chain c draws from make_rng(seed, c) whichever rank owns it."""
    one = chain_rngs(5, shard_chains(6, 1, 0))
    two = chain_rngs(5, shard_chains(6, 2, 1))
    a = [r.standard_normal(4) for r in one][3:]
    b = [r.standard_normal(4) for r in two]
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = shard_chains(total, world, rank)
        chains = np.arange(shard.start, shard.stop, dtype=np.float64)
        local = {"dh": 0.01 * chains, "accepted": (chains % 3 != 0).astype(np.float64),
                 "chain": chains}
        got = gather_observables(local, shard)
        out_q.put((rank, {k: v.tolist() for k, v in got.items()}))
    finally:
        dist.destroy_process_group()


def _dd_worker(rank, world, port, L, T, out_q):
    """Execute the NCCL face-exchange plan of csrc/dd.cu (dd.halo_plan) with
    gloo point-to-point on CPU tensors and check every halo row."""
    import torch
    from paper_1512_03812_b200.dd import HALO, halo_plan
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lloc = L // world
        full = torch.arange(L * T, dtype=torch.float64).reshape(L, T)
        ext = torch.full((lloc + 2 * HALO, T), -1.0)
        ext[HALO:HALO + lloc] = full[rank * lloc:(rank + 1) * lloc]
        ops = []
        for peer, row, n, kind in halo_plan(rank, world, lloc):
            buf = ext[row:row + n]
            if kind == "send":
                ops.append(dist.P2POp(dist.isend, buf.contiguous(), peer))
            else:
                ops.append(dist.P2POp(dist.irecv, buf, peer))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        rows = (rank * lloc + np.arange(-HALO, lloc + HALO)) % L
        out_q.put((rank, bool(torch.equal(ext, full[torch.as_tensor(rows)]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dd_halo_plan_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dd_worker, args=(r, world, port, 12, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(res.values()), res


@pytest.mark.parametrize("total", [7, 64])
def test_gather_observables_world2_gloo(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(2):
        obs = {k: np.array(v) for k, v in res[rank].items()}
        assert np.array_equal(obs["chain"], np.arange(total))
        assert np.allclose(obs["dh"], 0.01 * np.arange(total))
        s = summarize(obs)
        assert abs(s["acceptance"] - np.mean(np.arange(total) % 3 != 0)) < 1e-15


def _handles_worker(rank, world, port, out_q):
    from paper_1512_03812_b200.dd import IPC_HANDLE_BYTES, allgather_handles
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank + 1]) * IPC_HANDLE_BYTES
        out_q.put((rank, allgather_handles(mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_p2p_ipc_handles_allgather_rank_order_gloo(world):
    """The p2p transport's one host-side collective: every rank ends up with
    all mailbox handles in rank order (the layout sch_dd_p2p_connect maps)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_handles_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = b"".join(bytes([r + 1]) * 64 for r in range(world))
    assert all(v == want for v in res.values())
