"""The device replica of the reference's NumPy streams (§8(f) row 2):
value-identical draws to make_rng(seed, stream) for every distribution the
HMC path uses, and a device-RNG ensemble that reproduces independent
reference chains trajectory by trajectory."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_standard_normal_stream_is_bit_identical():
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=20240401, n_chains=5, stream0=3)
    got = g.standard_normal((200_000,)).cpu().numpy()    # exercises the ziggurat tail/wedges
    for c in range(5):
        ref = sw.make_rng(20240401, 3 + c).standard_normal(200_000)
        assert np.array_equal(got[c], ref), c
    # the stream continues where it left off
    more = g.standard_normal((7,)).cpu().numpy()
    r = sw.make_rng(20240401, 3)
    r.standard_normal(200_000)
    assert np.array_equal(more[0], r.standard_normal(7))


def test_uniform_random_and_hot_start_are_bit_identical():
    import paper_1512_03812_b200 as sw
    geom = sw.LatticeGeom(6, 10)
    g = sw.NumpyDeviceRng(seed=7, n_chains=3)
    hs = g.hot_start(geom).cpu().numpy()
    u = g.random().cpu().numpy()
    w = g.uniform(-2.5, 4.0, (33,)).cpu().numpy()
    for c in range(3):
        r = sw.make_rng(7, c)
        assert np.array_equal(hs[c], r.uniform(-np.pi, np.pi, size=(2, 6, 10)))
        assert u[c] == r.random()
        assert np.array_equal(w[c], r.uniform(-2.5, 4.0, size=33))


def test_heatbath_draws_match_reference_order():
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.fermion import draw_phi
    geom = sw.LatticeGeom(8, 4)
    g = sw.NumpyDeviceRng(seed=11, n_chains=4)
    p, phi = g.heatbath(geom)
    for c in range(4):
        r = sw.make_rng(11, c)
        assert np.array_equal(p[c].cpu().numpy(), r.standard_normal((2, 8, 4)))
        assert np.array_equal(phi[c].cpu().numpy(), draw_phi(r, 8, 4))


def test_metropolis_draws_only_uphill():
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=3, n_chains=4)
    dh = torch.tensor([-0.5, 0.7, 0.0, float("nan")], dtype=torch.float64, device="cuda")
    acc = g.metropolis(dh).cpu().numpy()
    follow = g.random().cpu().numpy()
    for c, d in enumerate([-0.5, 0.7, 0.0]):
        r = sw.make_rng(3, c)
        want = sw.metropolis(d, r)
        assert acc[c] == int(want)
        assert follow[c] == r.random()      # exactly one draw consumed iff dH > 0
    assert acc[3] == -1


def test_device_stream_ensemble_matches_reference_chains():
    """Hot start + 3 trajectories per chain on device streams == the same
    chains run by the CPU oracle with make_rng(seed, c): dH <= 1e-8, same
    accept sequence."""
    import paper_1512_03812_b200 as sw
    from oracle import schwinger_oracle as O
    B, L = 3, 8
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    ocfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                    micro_per_call=2, cg_tol=1e-10)
    g = sw.NumpyDeviceRng(seed=99, n_chains=B)
    q = g.hot_start(sw.LatticeGeom(L, L))
    rngs = [O.make_rng(99, c) for c in range(B)]
    qo = np.stack([O.hot_start(r, L, L) for r in rngs])
    assert np.array_equal(q.cpu().numpy(), qo)
    for _ in range(3):
        q, st = sw.hmc_update_ensemble(q, cfg, device_rng=g)
        qo, so = O.ensemble_update(qo, ocfg, rngs)
        assert np.max(np.abs(st.dh - np.array([s["dh"] for s in so]))) < 1e-8
        assert np.array_equal(st.accepted, np.array([s["accepted"] for s in so]))
    assert np.max(np.abs(q.cpu().numpy() - qo)) < 1e-8


def test_rng_state_export_continues_on_host():
    """get_states() are NumPy Philox states: a host Generator built from one
    continues the device stream draw for draw (checkpoint / hand-back)."""
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=99, n_chains=4, stream0=10)
    g.standard_normal((1001,))   # odd count: leaves a partly used buffer
    g.random()
    states = g.get_states()
    dev = g.standard_normal((513,)).cpu().numpy()
    for c in range(4):
        ref = sw.make_rng(99, 10 + c)
        ref.standard_normal(1001)
        ref.random()
        assert states[c]["buffer_pos"] == ref.bit_generator.state["buffer_pos"]
        assert np.array_equal(states[c]["state"]["counter"], ref.bit_generator.state["state"]["counter"])
        h = np.random.Generator(np.random.Philox(key=[0, 0]))
        h.bit_generator.state = states[c]
        assert np.array_equal(h.standard_normal(513), dev[c])


def test_rng_from_host_generators_and_npz_checkpoint(tmp_path):
    import paper_1512_03812_b200 as sw
    gens = [sw.make_rng(5, s) for s in (3, 8, 21)]
    for i, h in enumerate(gens):   # advance each host stream differently
        h.standard_normal(17 * (i + 1))
        h.uniform(-1.0, 1.0, size=i)
    d = sw.NumpyDeviceRng.from_generators(gens)
    a = d.standard_normal((64,)).cpu().numpy()
    d.save(tmp_path / "rng.npz")
    b = d.uniform(-np.pi, np.pi, (40,)).cpu().numpy()
    d2 = sw.NumpyDeviceRng.load(tmp_path / "rng.npz")
    b2 = d2.uniform(-np.pi, np.pi, (40,)).cpu().numpy()
    assert np.array_equal(b, b2)
    for c, h in enumerate(gens):
        assert np.array_equal(a[c], h.standard_normal(64))
        assert np.array_equal(b[c], h.uniform(-np.pi, np.pi, size=40))
    with pytest.raises(ValueError):
        d.set_states(d.get_states()[:2])


def test_ensemble_checkpoint_resume_and_hand_back_to_reference(tmp_path):
    """save_checkpoint after 2 device trajectories; resuming it on the GPU is
    bit-identical to the uninterrupted run, and the same file loaded with host
    generators continues chain by chain in the CPU oracle (dH <= 1e-8, same
    accept sequence)."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200 import ensemble as E
    from oracle import schwinger_oracle as O
    B, L = 3, 8
    cfg = sw.HmcConfig(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                       micro_per_call=2, cg_tol=1e-10)
    ocfg = O.Config(L=L, T=L, beta=2.0, m0=0.1, tau=1.0, h=1.0 / 3.0, scheme="adapted-nested-fg",
                    micro_per_call=2, cg_tol=1e-10)
    g = sw.NumpyDeviceRng(seed=4242, n_chains=B)
    q = g.hot_start(sw.LatticeGeom(L, L))
    for _ in range(2):
        q, _ = sw.hmc_update_ensemble(q, cfg, device_rng=g)
    E.save_checkpoint(tmp_path / "ck.npz", q, g, trajectory=2, meta={"beta": 2.0})
    qa = q
    dha = []
    for _ in range(2):
        qa, st = sw.hmc_update_ensemble(qa, cfg, device_rng=g)
        dha.append(st.dh)
    qb, gb, shard, traj, meta = E.load_checkpoint(tmp_path / "ck.npz")
    assert traj == 2 and meta == {"beta": 2.0} and shard.count == B
    for k in range(2):
        qb, st = sw.hmc_update_ensemble(qb, cfg, device_rng=gb)
        assert np.array_equal(st.dh, dha[k])
    assert torch.equal(qa, qb)
    qo, rngs, _, _, _ = E.load_checkpoint(tmp_path / "ck.npz", device_rng=False)
    qo = qo.cpu().numpy()
    for k in range(2):
        qo, so = O.ensemble_update(qo, ocfg, rngs)
        assert np.max(np.abs(dha[k] - np.array([s["dh"] for s in so]))) < 1e-8
    assert np.max(np.abs(qa.cpu().numpy() - qo)) < 1e-8


def test_long_stream_parallel_walk_is_bit_identical():
    """A few long streams are walked by the whole GPU (csrc/nprng.cu: chunks
    of 2048 words counted, scanned with the ~1 % of entry-offset corrections,
    then emitted): 3 M normals of one stream — wedges, tails, passes that run
    across chunk ends — are NumPy's bit for bit, from a state that starts in
    the middle of a Philox block, and the stream continues on the serial path."""
    import paper_1512_03812_b200 as sw
    g = sw.NumpyDeviceRng(seed=99, n_chains=1, stream0=4)
    r = sw.make_rng(99, 4)
    assert np.array_equal(g.uniform(0.0, 1.0, (3,)).cpu().numpy()[0], r.uniform(0.0, 1.0, size=3))
    n = 3_000_000
    got = g.standard_normal((n,)).cpu().numpy()[0]
    assert np.array_equal(got, r.standard_normal(n))
    assert np.array_equal(g.standard_normal((11,)).cpu().numpy()[0], r.standard_normal(11))
    assert g.random().cpu().numpy()[0] == r.random()
    # uniforms of a long stream (a thread per Philox block), then normals again
    assert np.array_equal(g.uniform(-np.pi, np.pi, (2, 300, 301)).cpu().numpy()[0],
                          r.uniform(-np.pi, np.pi, size=(2, 300, 301)))
    assert np.array_equal(g.uniform(0.0, 1.0, (131_073,)).cpu().numpy()[0], r.uniform(0.0, 1.0, size=131_073))
    assert g.random().cpu().numpy()[0] == r.random()
    # a length just above the threshold of the parallel path, twice in a row
    for m in (131_072, 140_001):
        assert np.array_equal(g.standard_normal((m,)).cpu().numpy()[0], r.standard_normal(m)), m


@pytest.mark.parametrize("quenched", [False, True])
def test_long_stream_heatbath_matches_reference_order(quenched):
    """The decomposed lattice's heatbath: p, Re phi, Im phi of a 256 x 256
    lattice from one stream through the parallel walk (393 k normals), then
    the Metropolis uniform from the state it leaves."""
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200.fermion import draw_phi
    L = 256
    geom = sw.LatticeGeom(L, L)
    g = sw.NumpyDeviceRng(seed=5, n_chains=2, stream0=0)
    p, phi = g.heatbath(geom, quenched=quenched)
    u = g.random().cpu().numpy()
    for c in range(2):
        r = sw.make_rng(5, c)
        assert np.array_equal(p[c].cpu().numpy(), r.standard_normal((2, L, L)))
        if not quenched:
            assert np.array_equal(phi[c].cpu().numpy(), draw_phi(r, L, L))
        assert u[c] == r.random()


_PAR_SNIPPET = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_1512_03812_b200 as sw
g = sw.NumpyDeviceRng(seed=31, n_chains=3, stream0=9)
out = {"u": g.uniform(0.0, 1.0, (2,)).cpu().numpy(),
       "hs": g.hot_start(sw.LatticeGeom(300, 256)).cpu().numpy(),
       "a": g.standard_normal((700_001,)).cpu().numpy(),
       "b": g.standard_normal((150_000,)).cpu().numpy()}
p, phi = g.heatbath(sw.LatticeGeom(192, 384))
out["p"], out["phi"] = p.cpu().numpy(), phi.cpu().numpy()
out["tail"] = g.standard_normal((5,)).cpu().numpy()
out["state"] = np.frombuffer(g.state.cpu().numpy().tobytes(), dtype=np.uint8)
np.savez(sys.argv[2], **out)
"""


def test_long_stream_parallel_walk_equals_serial_walk(tmp_path):
    """The whole-GPU walk of a long stream against the warp-per-stream walk
    (SCH_NP_PAR=0) on the same draws: values and the generator state left
    behind, byte for byte — with the production chunk of 2048 words and with
    chunks of 7 and 33 words (SCH_NP_CHUNK), where most chunks are entered at
    an offset, slow passes straddle chunk ends and a tail pass can swallow a
    whole chunk.  The switches are read once per process."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    res = {}
    for name, env in (("serial", {"SCH_NP_PAR": "0"}), ("par", {}), ("par7", {"SCH_NP_CHUNK": "7"}),
                      ("par33", {"SCH_NP_CHUNK": "33"})):
        path = tmp_path / f"{name}.npz"
        subprocess.run([sys.executable, "-c", _PAR_SNIPPET, root, str(path)], check=True,
                       env=dict(os.environ, **env), timeout=600)
        res[name] = np.load(path)
    for name in ("par", "par7", "par33"):
        for k in res["serial"].files:
            assert np.array_equal(res["serial"][k], res[name][k]), (name, k)
