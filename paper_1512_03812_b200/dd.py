"""One large lattice decomposed into x-strips (BASELINE configs[4], SURVEY
§8(e) mode 2): D^dag D and CG with halo exchange and global reductions.

The lattice's L rows are split into G strips of Lloc = L/G rows.  Each strip
is stored as an *extended strip* of Lext = Lloc + 4 rows (two halo rows per
side, enough for the fused D^dag D).  Two transports share one code path in
the C library (csrc/dd.cu):

* local — ``StripLattice(L, T, strips=G)`` keeps every strip in this process
  as a batch (shape ``(G, Lext, T, ...)``); the halo exchange is a copy
  kernel.  This is how the decomposed path is exercised on one GPU.
* NCCL — ``StripLattice(L, T, group=pg)`` under ``torch.distributed`` with one
  strip per rank; faces go over ``ncclSend/ncclRecv`` to the +-x neighbour
  ranks and the CG scalars over ``ncclAllReduce``.
* p2p — ``transport="p2p"``: peer-memory mailboxes (csrc/dd.cu): push kernels
  store faces and reduction partials straight into the neighbours' HBM over
  NVLink (CUDA IPC mappings exchanged once through ``torch.distributed``),
  pull / finish kernels wait on release/acquire counters.  With every strip
  in one process (``strips=G``) the same kernels run on local mailboxes.

The periodic stencil kernels run unchanged on the extended strip; rows
outside the own range are masked out of outputs and reductions.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .fermion import FERMION_BC, SolverError
from .lattice import as_links, as_spinor

HALO = 2


def halo_plan(rank: int, world: int, lloc: int):
    """Face transfers of one exchange for one strip: (peer, first_row, nrows,
    direction) with direction 'send'/'recv', rows in extended-strip numbering
    (what csrc/dd.cu issues as grouped ncclSend/ncclRecv)."""
    left, right = (rank - 1) % world, (rank + 1) % world
    return [(right, lloc, 2, "send"), (left, 0, 2, "recv"),
            (left, 2, 2, "send"), (right, lloc + 2, 2, "recv")]


IPC_HANDLE_BYTES = 64


def allgather_handles(handle: bytes, group=None) -> bytes:
    """Every rank's 64-byte mailbox handle, concatenated in rank order (what
    sch_dd_p2p_connect takes)."""
    if len(handle) != IPC_HANDLE_BYTES:
        raise ValueError(f"IPC handle must be {IPC_HANDLE_BYTES} bytes, got {len(handle)}")
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return bytes(handle)
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return b"".join(out)


TRANSPORTS = ("local", "nccl", "p2p")


class StripLattice:
    """Geometry + C-side handle of an L x T lattice split into x-strips.

    ``transport``: "local" (all strips here, copy-kernel halos), "nccl" (one
    strip per rank) or "p2p" (peer-memory mailboxes; one strip per rank, or
    all strips here).  Default: "nccl" under a multi-rank process group,
    else "local"."""

    def __init__(self, L: int, T: int, strips: int | None = None, group=None,
                 transport: str | None = None):
        self.L, self.T = int(L), int(T)
        multi = group is not None or (strips is None and dist.is_initialized()
                                      and dist.get_world_size() > 1)
        if transport is None:
            transport = "nccl" if multi else "local"
        if transport not in TRANSPORTS:
            raise ValueError(f"unknown transport {transport!r}; valid: {', '.join(TRANSPORTS)}")
        if transport == "nccl" and not (multi or (group is None and strips is None
                                                  and dist.is_initialized())):
            raise ValueError("the NCCL transport needs a torch.distributed process group")
        if transport == "nccl":
            multi = True   # one strip per rank, even on a one-rank group
        if transport == "local" and multi:
            raise ValueError("the local transport keeps every strip in one process")
        self.transport = transport
        self.group = group   # every collective of this lattice runs on it (None: the default group)
        if multi:
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            self.local = 1
        else:
            self.world, self.rank, self.local = 1, 0, int(strips or 1)
        ctx = _lib.ctx()
        nid = None
        if transport == "nccl":
            buf = ctypes.create_string_buffer(128)
            if self.rank == 0:
                ctx.call("sch_nccl_unique_id", ctypes.cast(buf, ctypes.c_void_p))
            obj = [bytes(buf.raw)]
            src = 0 if group is None else dist.get_global_rank(group, 0)   # the group's rank 0
            dist.broadcast_object_list(obj, src=src, group=group)
            nid = ctypes.create_string_buffer(obj[0], 128)
        handle = ctypes.c_void_p()
        ctx.call("sch_dd_create", None if nid is None else ctypes.cast(nid, ctypes.c_void_p),
                 self.world, self.rank, self.L, self.T, self.local, ctypes.byref(handle))
        self._handle = handle
        geo = (ctypes.c_int * 4)()
        _lib.load().sch_dd_geometry(handle, geo)
        self.S, self.Lloc, self.Lext, self.G = (int(v) for v in geo)
        self.strip0 = self.rank * self.local     # global index of the first local strip
        if transport == "p2p":
            h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
            ctx.call("sch_dd_p2p_open", handle, ctypes.cast(h, ctypes.c_void_p))
            if self.world > 1:
                dist.barrier(group=group)   # every mailbox zeroed before anyone maps it
            allh = allgather_handles(h.raw, group)
            buf = ctypes.create_string_buffer(allh, len(allh))
            ctx.call("sch_dd_p2p_connect", handle, ctypes.cast(buf, ctypes.c_void_p))

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                _lib.load().sch_dd_destroy(h)
            except Exception:
                pass

    # -- layout helpers (host/torch plumbing, used by tests and setup) -----
    def _rows(self, g: int) -> np.ndarray:
        """Global rows of extended strip g (periodic)."""
        return (g * self.Lloc + np.arange(-HALO, self.Lloc + HALO)) % self.L

    def scatter_links(self, q) -> torch.Tensor:
        """(2, L, T) -> local extended strips (S, 2, Lext, T), halos filled."""
        q = as_links(q)
        idx = [torch.as_tensor(self._rows(self.strip0 + s), device=q.device) for s in range(self.S)]
        return torch.stack([q[:, i, :] for i in idx]).contiguous()

    def scatter_spinor(self, psi) -> torch.Tensor:
        """(L, T, 2) -> (S, Lext, T, 2), halos filled."""
        psi = as_spinor(psi)
        idx = [torch.as_tensor(self._rows(self.strip0 + s), device=psi.device) for s in range(self.S)]
        return torch.stack([psi[i] for i in idx]).contiguous()

    def own(self, ext: torch.Tensor, axis: int) -> torch.Tensor:
        """Own rows of an extended field along the x axis ``axis``."""
        return ext.narrow(axis, HALO, self.Lloc)

    def gather_links(self, ext) -> torch.Tensor:
        """(S, 2, Lext, T) -> own rows (2, S*Lloc, T) in global row order."""
        return torch.cat([ext[s][:, HALO:HALO + self.Lloc] for s in range(self.S)], dim=1)

    def gather_spinor(self, ext) -> torch.Tensor:
        """Local strips' own rows, concatenated in global row order."""
        return torch.cat([self.own(ext[s], 0) for s in range(self.S)], dim=0)

    def exchange(self, field: torch.Tensor, planes: int, words_per_site: int):
        _lib.ctx().call("sch_dd_exchange", self._handle, _lib.ptr(field), planes, words_per_site)
        return field


class DDWilsonDirac:
    """Wilson-Dirac operator on a decomposed lattice (fermion.py:88-131)."""

    def __init__(self, lattice: StripLattice, q_ext, m0: float, fermion_bc: str = "periodic"):
        self.lat = lattice
        self.q = as_links(q_ext)
        self.m0 = float(m0)
        self.U = torch.empty(self.q.shape, dtype=torch.complex128, device=self.q.device)
        # each extended strip is a Lext x T lattice for the link cache
        _lib.ctx().call("sch_links_to_u", _lib.ptr(self.q), _lib.ptr(self.U), lattice.S,
                        lattice.Lext, lattice.T, FERMION_BC[fermion_bc])

    def normal(self, psi_ext) -> torch.Tensor:
        """D^dag D on the own rows (halo rows of the output are not written)."""
        psi = as_spinor(psi_ext)
        out = torch.empty_like(psi)   # own rows written by the kernel, halo rows zeroed here
        out[:, :HALO].zero_()
        out[:, HALO + self.lat.Lloc:].zero_()
        _lib.ctx().call("sch_dd_ddagd", self.lat._handle, _lib.ptr(self.U), _lib.ptr(psi),
                        _lib.ptr(out), self.m0)
        return out

    def cg(self, b_ext, tol: float, maxiter: int = 10_000, x0_ext=None):
        """cg_normal on the decomposed lattice; returns (x_ext, iterations,
        relative residual) and raises SolverError at the cap."""
        b = as_spinor(b_ext).clone()
        x = torch.empty_like(b)
        x0 = None if x0_ext is None else as_spinor(x0_ext).clone()
        it, rel, st = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        rc = _lib.ctx().call("sch_dd_cg_normal", self.lat._handle, _lib.ptr(self.U), _lib.ptr(b),
                             _lib.ptr(x), _lib.ptr(x0), self.m0, float(tol), int(maxiter),
                             ctypes.byref(it), ctypes.byref(rel), ctypes.byref(st))
        if rc == _lib.SCH_ERR_SOLVER or st.value:
            raise SolverError(f"CG exceeded {maxiter} iterations", rel.value)
        return x, it.value, rel.value
