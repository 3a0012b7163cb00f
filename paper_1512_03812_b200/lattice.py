"""Geometry, RNG streams, link/momentum updates and gauge-config I/O.

Mirror of the reference ``schwinger.lattice`` (pkg/src/schwinger/lattice.py)
with fields resident on the B200: link-type fields are float64 CUDA tensors
of shape (..., 2, L, T), spinors complex128 CUDA tensors (..., L, T, 2) —
the reference's own layouts (lattice.py:3-12), so no conversion happens at
the boundary.  Every arithmetic operation runs in the sm_100a library; torch
only allocates and moves memory.

Random draws keep the reference convention (NumPy Philox keyed by
[seed, stream], lattice.py:86-89) and are drawn on the host in the
reference's order, then uploaded ("parity mode").  ``DeviceRng`` is the
bench-mode alternative that draws on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

TWO_PI = 2.0 * np.pi

LINK_X, LINK_T = -2, -1
SPIN_X, SPIN_T = -3, -2


# ---------------------------------------------------------------------------
# tensor plumbing
# ---------------------------------------------------------------------------

def device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def as_links(a) -> torch.Tensor:
    """float64 CUDA tensor (..., 2, L, T), contiguous."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return t.to(device=device(), dtype=torch.float64).contiguous()


def as_spinor(a) -> torch.Tensor:
    """complex128 CUDA tensor (..., L, T, 2), contiguous."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128))
    return t.to(device=device(), dtype=torch.complex128).contiguous()


def to_numpy(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return np.asarray(t)


def n_chains(t: torch.Tensor, core_dims: int = 3) -> int:
    """Number of chains in the leading batch dims (1 for an unbatched field)."""
    b = 1
    for d in t.shape[:-core_dims]:
        b *= d
    return b


def squeeze_chain(v: torch.Tensor, like: torch.Tensor, core_dims: int = 3) -> torch.Tensor:
    """Shape a per-chain vector (B,) like the batch dims of ``like`` (0-d if unbatched)."""
    return v.reshape(like.shape[:-core_dims])


def wrap_angles(q):
    """Reduce angles to [-pi, pi) (lattice.py:28-30)."""
    q = as_links(q)
    out = torch.empty_like(q)
    _lib.ctx().call("sch_wrap_angles", _lib.ptr(q), _lib.ptr(out), q.numel())
    return out


@dataclass(frozen=True)
class LatticeGeom:
    """Lattice extents, L sites in space and T in time (lattice.py:33-74)."""

    L: int
    T: int

    def __post_init__(self):
        if self.L < 2 or self.T < 2:
            raise ValueError(f"hopping stencils need L, T >= 2, got {self.L}x{self.T}")

    @property
    def volume(self) -> int:
        return self.L * self.T

    @property
    def n_links(self) -> int:
        return 2 * self.volume

    def site_index(self, x: int, t: int) -> int:
        return t * self.L + x

    def site_coords(self, idx: int) -> tuple[int, int]:
        return idx % self.L, idx // self.L

    def shift_site(self, site, mu: int, s: int):
        x, t = site
        if mu == 0:
            return (x + s) % self.L, t
        if mu == 1:
            return x, (t + s) % self.T
        raise ValueError(f"direction must be 0 or 1, got {mu}")

    def links_shape(self, batch: int | None = None):
        return (2, self.L, self.T) if batch is None else (batch, 2, self.L, self.T)

    def spinor_shape(self, batch: int | None = None):
        return (self.L, self.T, 2) if batch is None else (batch, self.L, self.T, 2)


def geom_of(field) -> LatticeGeom:
    return LatticeGeom(int(field.shape[-2]), int(field.shape[-1]))


# ---------------------------------------------------------------------------
# random streams (host, reference convention)
# ---------------------------------------------------------------------------

def make_rng(seed: int, stream: int = 0) -> np.random.Generator:
    """Counter-based generator keyed by [seed, stream] (lattice.py:86-89)."""
    key = np.array([seed % 2**64, stream % 2**64], dtype=np.uint64)
    return np.random.Generator(np.random.Philox(key=key))


def sample_momenta(rng, geom: LatticeGeom, batch: int | None = None) -> torch.Tensor:
    """Gaussian momenta, drawn with the reference generator (lattice.py:92-95)."""
    return as_links(rng.standard_normal(geom.links_shape(batch)))


def cold_start(geom: LatticeGeom, batch: int | None = None) -> torch.Tensor:
    return torch.zeros(geom.links_shape(batch), dtype=torch.float64, device=device())


def hot_start(rng, geom: LatticeGeom, batch: int | None = None) -> torch.Tensor:
    """theta ~ U(-pi, pi) (lattice.py:102-104)."""
    return as_links(rng.uniform(-np.pi, np.pi, size=geom.links_shape(batch)))


class DeviceRng:
    """Bench-mode generator: Philox4x32-10 on the GPU, one stream per chain
    (key = (seed, stream0 + chain)), advancing a per-draw counter.  Not
    value-identical to the reference's NumPy stream."""

    def __init__(self, seed: int, stream0: int = 0):
        self.seed = int(seed) % 2**64
        self.stream0 = int(stream0) % 2**64
        self.counter = 0

    def normal(self, n_chains: int, shape, scale: float = 1.0) -> torch.Tensor:
        out = torch.empty((n_chains,) + tuple(shape), dtype=torch.float64, device=device())
        per = out.numel() // n_chains
        _lib.ctx().call("sch_rng_normal", _lib.ptr(out), n_chains, per, self.seed, self.stream0,
                        self.counter, float(scale))
        self.counter += 1
        return out

    def complex_normal(self, n_chains: int, shape, scale: float) -> torch.Tensor:
        """complex128 field whose re/im parts are iid scale*N(0,1)."""
        out = torch.empty((n_chains,) + tuple(shape), dtype=torch.complex128, device=device())
        per = 2 * (out.numel() // n_chains)
        _lib.ctx().call("sch_rng_normal", _lib.ptr(out), n_chains, per, self.seed, self.stream0,
                        self.counter, float(scale))
        self.counter += 1
        return out

    def uniform(self, n_chains: int) -> torch.Tensor:
        out = torch.empty((n_chains,), dtype=torch.float64, device=device())
        _lib.ctx().call("sch_rng_uniform", _lib.ptr(out), n_chains, 1, self.seed, self.stream0,
                        self.counter)
        self.counter += 1
        return out


class NumpyDeviceRng:
    """Device replica of B reference streams: chain c draws exactly what
    ``make_rng(seed, stream0 + c)`` would (lattice.py:86-89) — same Philox4x64
    counter walk, same ziggurat normals, same uniform/random doubles — with the
    state kept on the GPU.  Lets device-side ensembles (bench mode) keep
    value-level parity with the reference's per-chain trajectories."""

    def __init__(self, seed: int, n_chains: int, stream0: int = 0):
        lib = _lib.load()
        self.n = int(n_chains)
        self.seed, self.stream0 = int(seed) % 2**64, int(stream0) % 2**64
        nbytes = int(lib.sch_np_rng_state_bytes())
        if nbytes != _NP_STATE_DTYPE.itemsize:
            raise _lib.NativeUnavailable(f"device RNG state is {nbytes} B, host expects 88")
        self.state = torch.empty((self.n * nbytes,), dtype=torch.uint8, device=device())
        _lib.ctx().call("sch_np_rng_init", _lib.ptr(self.state), self.n, self.seed, self.stream0)

    def _fill(self, shape, mode, lo=0.0, hi=0.0) -> torch.Tensor:
        out = torch.empty((self.n,) + tuple(shape), dtype=torch.float64, device=device())
        per = out.numel() // self.n
        _lib.ctx().call("sch_np_rng_fill", _lib.ptr(self.state), _lib.ptr(out), self.n, per, mode,
                        float(lo), float(hi))
        return out

    def standard_normal(self, shape) -> torch.Tensor:
        return self._fill(shape, 0)

    def uniform(self, low: float, high: float, shape) -> torch.Tensor:
        return self._fill(shape, 1, low, high)

    def random(self) -> torch.Tensor:
        return self._fill((), 2).reshape(self.n)

    def hot_start(self, geom: LatticeGeom) -> torch.Tensor:
        """theta ~ U(-pi, pi) per chain (lattice.py:102-104)."""
        return self.uniform(-np.pi, np.pi, geom.links_shape())

    def heatbath(self, geom: LatticeGeom, quenched: bool = False):
        """(p, phi) of hmc_update's draws, reference order (hmc.py:78-82)."""
        p = torch.empty((self.n,) + geom.links_shape(), dtype=torch.float64, device=device())
        phi = None if quenched else torch.empty((self.n,) + geom.spinor_shape(),
                                                dtype=torch.complex128, device=device())
        scale = 1.0 / np.sqrt(2.0)   # NumPy divides the complex phi by sqrt(2) this way
        _lib.ctx().call("sch_np_heatbath", _lib.ptr(self.state), _lib.ptr(p), _lib.ptr(phi), self.n,
                        geom.volume, float(scale), int(quenched))
        return p, phi

    def metropolis(self, dh: torch.Tensor) -> torch.Tensor:
        """Accept flags (1/0, -1 for non-finite dH), one uniform iff dH > 0."""
        acc = torch.empty((self.n,), dtype=torch.int32, device=dh.device)
        _lib.ctx().call("sch_np_metropolis", _lib.ptr(self.state), _lib.ptr(dh), _lib.ptr(acc), self.n)
        return acc

    # -- checkpointing: the per-chain Philox counters ----
    # The device record is NumPy's own Philox state (counter[4], key[2],
    # buffer[4], buffer_pos), so a chain's stream can be handed to or taken
    # from a host np.random.Generator at any point and continue identically.

    def get_states(self) -> list[dict]:
        """Per-chain ``Generator.bit_generator.state`` dicts (Philox)."""
        rec = _np_state_records(self.state.cpu().numpy())
        out = []
        for c in range(self.n):
            out.append({"bit_generator": "Philox",
                        "state": {"counter": rec["ctr"][c].copy(), "key": rec["key"][c].copy()},
                        "buffer": rec["buf"][c].copy(), "buffer_pos": int(rec["pos"][c]),
                        "has_uint32": 0, "uinteger": 0})
        return out

    def set_states(self, states) -> None:
        """Load per-chain Philox state dicts (e.g. from reference Generators)."""
        if len(states) != self.n:
            raise ValueError(f"expected {self.n} states, got {len(states)}")
        raw = np.zeros(self.state.numel(), dtype=np.uint8)
        rec = _np_state_records(raw)
        for c, s in enumerate(states):
            if s.get("bit_generator") != "Philox":
                raise ValueError("only Philox generator states can be loaded")
            if s.get("has_uint32", 0):
                raise ValueError("a pending 32-bit half word cannot be carried over")
            rec["ctr"][c] = np.asarray(s["state"]["counter"], dtype=np.uint64)
            rec["key"][c] = np.asarray(s["state"]["key"], dtype=np.uint64)
            rec["buf"][c] = np.asarray(s["buffer"], dtype=np.uint64)
            pos = int(s["buffer_pos"])
            if not 0 <= pos <= 4:
                raise ValueError(f"buffer_pos {pos} out of range")
            rec["pos"][c] = pos
        self.state.copy_(torch.from_numpy(raw).to(self.state.device))

    @classmethod
    def from_generators(cls, gens) -> "NumpyDeviceRng":
        """Device streams continuing the given host Generators exactly."""
        gens = list(gens)
        self = cls(0, len(gens))
        self.set_states([g.bit_generator.state for g in gens])
        return self

    def save(self, path) -> None:
        """Write the per-chain counters/keys/buffers to an .npz checkpoint."""
        rec = _np_state_records(self.state.cpu().numpy())
        np.savez(path, ctr=rec["ctr"], key=rec["key"], buf=rec["buf"], pos=rec["pos"].astype(np.int32),
                 seed=np.uint64(self.seed), stream0=np.uint64(self.stream0))

    @classmethod
    def load(cls, path) -> "NumpyDeviceRng":
        z = np.load(path)
        n = int(z["ctr"].shape[0])
        self = cls(int(z["seed"]), n, int(z["stream0"]))
        self.set_states([{"bit_generator": "Philox",
                          "state": {"counter": z["ctr"][c], "key": z["key"][c]},
                          "buffer": z["buf"][c], "buffer_pos": int(z["pos"][c])}
                         for c in range(n)])
        return self


_NP_STATE_DTYPE = np.dtype([("ctr", "<u8", (4,)), ("key", "<u8", (2,)), ("buf", "<u8", (4,)),
                            ("pos", "<i4"), ("pad", "<i4")])   # csrc/nprng.cu NpPhilox (88 B)


def _np_state_records(raw: np.ndarray) -> np.ndarray:
    """View a device-state byte image as NpPhilox records (no copy)."""
    assert _NP_STATE_DTYPE.itemsize == 88
    return raw.view(_NP_STATE_DTYPE)


# ---------------------------------------------------------------------------
# elementary updates (device)
# ---------------------------------------------------------------------------

def rotate_links(q, p, h: float) -> torch.Tensor:
    """Group-exact drift q -> wrap(q + h p) (lattice.py:111-118)."""
    q, p = as_links(q), as_links(p)
    if q.shape != p.shape:
        q, p = torch.broadcast_tensors(q, p)
        q, p = q.contiguous(), p.contiguous()
    out = torch.empty_like(q)
    _lib.ctx().call("sch_rotate_links", _lib.ptr(q), _lib.ptr(p), float(h), _lib.ptr(out), q.numel())
    return out


def shift_momenta(p, force, h: float) -> torch.Tensor:
    """p -> p - h*force (lattice.py:121-125)."""
    p, force = as_links(p), as_links(force)
    if p.shape[-3:] != force.shape[-3:]:
        raise ValueError(f"shape mismatch: momenta {tuple(p.shape)} vs force {tuple(force.shape)}")
    return kick(p, force, h)


def kick(p: torch.Tensor, f: torch.Tensor, a: float, g: torch.Tensor | None = None,
         c: float = 0.0) -> torch.Tensor:
    """out = p - (a*f + c*g), or p - a*f without g (NumPy operation order)."""
    if p.shape != f.shape or (g is not None and g.shape != p.shape):
        shape = torch.broadcast_shapes(p.shape, f.shape, *(() if g is None else (g.shape,)))
        p = p.expand(shape).contiguous()
        f = f.expand(shape).contiguous()
        g = None if g is None else g.expand(shape).contiguous()
    out = torch.empty_like(p)
    _lib.ctx().call("sch_kick", _lib.ptr(p), _lib.ptr(f), float(a), _lib.ptr(g), float(c),
                    _lib.ptr(out), p.numel())
    return out


def kinetic_energy(p) -> torch.Tensor:
    """(1/2) sum p^2 per chain (lattice.py:128-130); 0-d for an unbatched field."""
    p = as_links(p)
    B = n_chains(p)
    out = torch.empty((B,), dtype=torch.float64, device=p.device)
    _lib.ctx().call("sch_kinetic_energy", _lib.ptr(p), _lib.ptr(out), B, p.numel() // B)
    return squeeze_chain(out, p)


# ---------------------------------------------------------------------------
# gauge configuration files (lattice.py:137-172 format)
# ---------------------------------------------------------------------------

_MAGIC = "schwinger-u1 v1"


def save_gauge_config(path, q, beta: float, m0: float, seed: int) -> None:
    """ASCII header + 2V little-endian float64, site-major (t-major), directions
    interleaved; bit-exact round trip (lattice.py:140-154)."""
    q = to_numpy(q)
    if q.ndim != 3:
        raise ValueError("config files hold a single (2, L, T) configuration")
    g = geom_of(q)
    head = f"{_MAGIC} {g.L} {g.T} {beta!r} {m0!r} {seed}\n".encode("ascii")
    body = np.ascontiguousarray(np.transpose(q, (2, 1, 0)), dtype="<f8").tobytes()
    with open(path, "wb") as fh:
        fh.write(head + body)


def load_gauge_config(path, to_device: bool = False):
    """Read a 'schwinger-u1 v1' file (lattice.py:157-172); host array by default."""
    with open(path, "rb") as fh:
        head = fh.readline().decode("ascii").strip()
        body = fh.read()
    parts = head.split()
    if len(parts) != 7 or " ".join(parts[:2]) != _MAGIC:
        raise ValueError(f"{path}: not a schwinger-u1 v1 configuration (header {head!r})")
    L, T = int(parts[2]), int(parts[3])
    meta = {"L": L, "T": T, "beta": float(parts[4]), "m0": float(parts[5]), "seed": int(parts[6])}
    if len(body) != 2 * L * T * 8:
        raise ValueError(f"{path}: expected {2 * L * T * 8} payload bytes, got {len(body)}")
    q = np.ascontiguousarray(np.frombuffer(body, dtype="<f8").reshape(T, L, 2).transpose(2, 1, 0))
    return (as_links(q) if to_device else q), meta
