"""Model check of the peer-memory (p2p) transport protocol of csrc/dd.cu.

The kernels k_p2p_push / k_p2p_pull / k_p2p_red_push / k_p2p_red_finish
synchronise G strips (ranks) through counters in each other's mailboxes.
This test restates their rules step by step — sequence numbers, slot =
seq % 2, arrival thresholds kP2PBlk * seq, credit thresholds
kP2PBlk * (seq - 2), strip-ordered sums — and runs many random
interleavings of G ranks, each executing its own stream of exchanges and
global sums in order (one CTA step at a time), checking that

  * no interleaving deadlocks (every rank finishes its program),
  * every pull copies exactly the neighbour's data of the same exchange
    (no slot is overwritten before it was consumed),
  * every global sum sees exactly the G contributions of the same sum and
    gives the same value on every rank.

The cross-GPU memory ordering itself (release/acquire at system scope) is
what the CUDA code provides; this checks the counting and slot logic on
which the transport's correctness rests.  (1-GPU pool: the kernels run on
the GPU only in loopback, tests/test_gpu_dd.py.)
"""

import random

import pytest

NBLK = 2    # CTAs per side of a push / pull launch (kP2PBlk in csrc/dd.cu, 16; the logic is per CTA)
NBUF = 2    # slots per side (kNBuf)


class Mailbox:
    def __init__(self, G):
        self.arrived = [0, 0]          # side 0: from the left neighbour, 1: from the right
        self.acked = [0, 0]            # credits for what this strip pushed right (0) / left (1)
        self.face = [[None] * NBUF for _ in range(2)]   # side x slot -> list of NBLK parts
        self.redflag = [0] * G
        self.red = [[None] * G for _ in range(NBUF)]


def kernel_steps(op, g, G, boxes, state, log):
    """Generator of the atomic steps of one kernel launch of rank g; yields
    False while blocked on a wait, True after progress."""
    kind = op[0]
    if kind == "push":
        seq = state["xseq"] + 1
        for d in (0, 1):                 # the two sides run as independent CTAs; model in order
            tgt = (g + 1) % G if d == 0 else (g - 1) % G
            for b in range(NBLK):
                while seq > NBUF and boxes[g].acked[d] < NBLK * (seq - NBUF):
                    yield False
                slot = boxes[tgt].face[d]
                if slot[seq % NBUF] is None or slot[seq % NBUF][0] != seq:
                    slot[seq % NBUF] = [seq, [None] * NBLK]
                slot[seq % NBUF][1][b] = ("face", g, seq, d, b)
                boxes[tgt].arrived[d] += 1
                yield True
    elif kind == "pull":
        seq = state["xseq"] + 1
        done = 0
        for d in (0, 1):
            src = (g - 1) % G if d == 0 else (g + 1) % G
            for b in range(NBLK):
                while boxes[g].arrived[d] < NBLK * seq:
                    yield False
                entry = boxes[g].face[d][seq % NBUF]
                got = entry[1]
                want = [("face", src, seq, d, k) for k in range(NBLK)]
                if entry[0] != seq or got != want:
                    log.append(f"rank {g} pull seq {seq} side {d}: got {entry}")
                boxes[src].acked[d] += 1
                done += 1
                yield True
        state["xseq"] = seq                # the last pull CTA advances the counter
    elif kind == "red_push":
        seq = state["rseq"] + 1
        val = op[1][g]
        for h in range(G):
            boxes[h].red[seq % NBUF][g] = (seq, val)
            yield True
        for h in range(G):
            boxes[h].redflag[g] = seq
            yield True
    elif kind == "red_finish":
        seq = state["rseq"] + 1
        for h in range(G):
            while boxes[g].redflag[h] < seq:
                yield False
        vals = []
        for h in range(G):
            s, v = boxes[g].red[seq % NBUF][h]
            if s != seq:
                log.append(f"rank {g} sum {seq}: slot {h} holds sum {s}")
            vals.append(v)
        total = 0.0
        for v in vals:                     # strip order
            total += v
        state["sums"].append(total)
        state["rseq"] = seq
        yield True


def program(rng, n_ops):
    """A rank's stream: exchanges (push, pull) and global sums (push,
    finish) in a random but common order; sum inputs differ per call."""
    ops = []
    for k in range(n_ops):
        if rng.random() < 0.5:
            ops += [("push",), ("pull",)]
        else:
            vals = [rng.random() for _ in range(8)]
            ops += [("red_push", vals), ("red_finish",)]
    return ops


def run(G, seed, n_ops=12):
    rng = random.Random(seed)
    prog = program(rng, n_ops)
    boxes = [Mailbox(G) for _ in range(G)]
    states = [{"xseq": 0, "rseq": 0, "sums": []} for _ in range(G)]
    pcs = [0] * G
    gens = [None] * G
    log = []
    stalls = 0
    while any(pc < len(prog) for pc in pcs):
        live = [g for g in range(G) if pcs[g] < len(prog)]
        g = rng.choice(live)
        if gens[g] is None:
            gens[g] = kernel_steps(prog[pcs[g]], g, G, boxes, states[g], log)
        try:
            progressed = next(gens[g])
        except StopIteration:
            gens[g] = None
            pcs[g] += 1
            stalls = 0
            continue
        stalls = 0 if progressed else stalls + 1
        if stalls > 20_000:   # nobody made progress for a long random schedule
            raise AssertionError(f"deadlock: pcs={pcs} ops={[prog[p][0] for p in pcs if p < len(prog)]}")
    assert not log, log[:3]
    sums = [s["sums"] for s in states]
    assert all(s == sums[0] for s in sums), "global sums differ between ranks"
    return states


@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_p2p_protocol_random_interleavings(G):
    for seed in range(60):
        run(G, seed)


def test_p2p_protocol_runs_ahead_without_sums():
    """A stream of exchanges with no global sum in between: only the credits
    keep a fast producer from overwriting unconsumed slots."""
    G = 3
    for seed in range(40):
        rng = random.Random(seed)
        boxes = [Mailbox(G) for _ in range(G)]
        states = [{"xseq": 0, "rseq": 0, "sums": []} for _ in range(G)]
        prog = [("push",), ("pull",)] * 9
        pcs, gens, log = [0] * G, [None] * G, []
        steps = 0
        while any(pc < len(prog) for pc in pcs):
            g = rng.choice([h for h in range(G) if pcs[h] < len(prog)])
            if gens[g] is None:
                gens[g] = kernel_steps(prog[pcs[g]], g, G, boxes, states[g], log)
            try:
                next(gens[g])
            except StopIteration:
                gens[g] = None
                pcs[g] += 1
            steps += 1
            assert steps < 200_000, "no progress"
        assert not log, log[:3]
