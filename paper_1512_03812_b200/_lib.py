"""ctypes binding of the sm_100a C-ABI (include/schwinger_sm100.h).

The shared library is built in-tree (``paper_1512_03812_b200/_lib/
libschwinger_sm100.so``) by ``__graft_entry__.build()`` / ``make -C
paper_1512_03812_b200/csrc``.  There is no CPU fallback: if the library or a
CUDA device is missing every operator raises ``NativeUnavailable``.

Device buffers are torch CUDA tensors (plumbing only); their ``data_ptr()`` is
handed to the C side together with the plain sizes.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libschwinger_sm100.so"

_c_int, _c_ll, _c_dbl, _c_ptr = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
_c_u64 = ctypes.c_uint64

# name -> argtypes (restype is int unless listed in _RESTYPES)
_SIGNATURES = {
    "sch_ctx_create": [_c_int, ctypes.POINTER(_c_ptr)],
    "sch_ctx_destroy": [_c_ptr],
    "sch_set_stream": [_c_ptr, _c_ptr],
    "sch_last_error": [_c_ptr],
    "sch_launch_count": [_c_ptr],
    "sch_build_info": [],
    "sch_rotate_links": [_c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_ll],
    "sch_wrap_angles": [_c_ptr, _c_ptr, _c_ptr, _c_ll],
    "sch_kick": [_c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_dbl, _c_ptr, _c_ll],
    "sch_kinetic_energy": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_ll],
    "sch_plaquette_angles": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int],
    "sch_gauge_force": [_c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_int, _c_int, _c_int],
    "sch_kick_gauge": [_c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_ptr, _c_int, _c_int, _c_int],
    "sch_inner_leapfrog": [_c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_int, _c_int, _c_int, _c_int],
    "sch_gauge_action": [_c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_int, _c_int, _c_int],
    "sch_avg_plaquette": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int],
    "sch_fg_gauge_gauge": [_c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_int, _c_int, _c_int],
    "sch_gauge_hessian_dot": [_c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_ptr, _c_int, _c_int, _c_int],
    "sch_plaquette_stencil": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_int],
    "sch_link_bilinears": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_ptr, _c_ptr, _c_int, _c_int,
                           _c_int],
    "sch_links_to_u": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_int],
    "sch_dslash": [_c_ptr, _c_ptr, _c_int, _c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_dbl, _c_int],
    "sch_ddagd": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_dbl],
    "sch_spinor_dot": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_ll],
    "sch_cg_normal": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_dbl,
                      _c_dbl, _c_int, _c_int, _c_ptr, _c_ptr, _c_ptr, ctypes.POINTER(_c_int)],
    "sch_fermion_force": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_int, _c_int],
    "sch_kick_fermion": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_ptr, _c_dbl, _c_ptr,
                         _c_int, _c_int, _c_int],
    "sch_weighted_w_sums": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_int,
                            _c_int],
    "sch_fg_fermion_combine": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr,
                               _c_int, _c_int, _c_int],
    "sch_rng_normal": [_c_ptr, _c_ptr, _c_int, _c_ll, _c_u64, _c_u64, _c_u64, _c_dbl],
    "sch_rng_uniform": [_c_ptr, _c_ptr, _c_int, _c_ll, _c_u64, _c_u64, _c_u64],
    "sch_select_chains": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_ll],
    "sch_metropolis": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int],
    "sch_probe_fp64": [_c_ptr, _c_ptr, _c_int, _c_int],
    "sch_np_rng_state_bytes": [],
    "sch_np_rng_init": [_c_ptr, _c_ptr, _c_int, _c_u64, _c_u64],
    "sch_np_rng_fill": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_ll, _c_int, _c_dbl, _c_dbl],
    "sch_np_heatbath": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int, _c_ll, _c_dbl, _c_int],
    "sch_np_metropolis": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_int],
    "sch_nccl_unique_id": [_c_ptr, _c_ptr],
    "sch_dd_create": [_c_ptr, _c_ptr, _c_int, _c_int, _c_int, _c_int, _c_int,
                      ctypes.POINTER(_c_ptr)],
    "sch_dd_destroy": [_c_ptr],
    "sch_dd_p2p_open": [_c_ptr, _c_ptr, _c_ptr],
    "sch_chi_xi": [_c_ptr] * 6 + [_c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_int, _c_int, _c_ptr,
                                  _c_ptr, _c_ptr],
    "sch_traj_anfg16": [_c_ptr] + [_c_ptr] * 7 + [_c_int, _c_dbl, _c_dbl, _c_dbl, _c_int, _c_dbl,
                                                 _c_dbl, _c_dbl, _c_dbl, _c_int, _c_int],
    "sch_dd_p2p_connect": [_c_ptr, _c_ptr, _c_ptr],
    "sch_dd_geometry": [_c_ptr, ctypes.POINTER(_c_int)],
    "sch_dd_exchange": [_c_ptr, _c_ptr, _c_ptr, _c_int, _c_int],
    "sch_dd_own_sum": [_c_ptr, _c_ptr, _c_int, _c_ptr, _c_ptr, _c_ptr],
    "sch_dd_ddagd": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_dbl],
    "sch_dd_cg_normal": [_c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_ptr, _c_dbl, _c_dbl, _c_int,
                         ctypes.POINTER(_c_int), ctypes.POINTER(_c_dbl), ctypes.POINTER(_c_int)],
}
_RESTYPES = {"sch_last_error": ctypes.c_char_p, "sch_launch_count": ctypes.c_ulonglong,
             "sch_build_info": ctypes.c_char_p}

SCH_ERR_SOLVER = 3


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device is missing: there is no fallback."""


_lock = threading.RLock()
_lib = None
_contexts: dict[tuple[int, int], "Context"] = {}


def load() -> ctypes.CDLL:
    """Load libschwinger_sm100.so and declare every exported symbol."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` or `make -C {LIB_PATH.parent.parent / 'csrc'}`")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, argtypes in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


class Context:
    """One sch_ctx per (CUDA device, stream): a context's workspace arena,
    graph cache and poll flag are only ever touched in its own stream's
    order, so work issued on different torch streams runs concurrently
    without sharing scratch memory."""

    def __init__(self, device: int, stream: int):
        lib = load()
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the B200 path has no CPU fallback")
        handle = _c_ptr()
        with torch.cuda.device(device):
            rc = lib.sch_ctx_create(device, ctypes.byref(handle))
        if rc != 0:
            raise NativeUnavailable(f"sch_ctx_create(device={device}) failed with status {rc} "
                                    "(is this an sm_100 GPU?)")
        self.lib = lib
        self.handle = handle
        self.device = device
        self.stream = stream
        lib.sch_set_stream(handle, _c_ptr(stream))

    def call(self, name: str, *args):
        rc = getattr(self.lib, name)(self.handle, *args)
        if rc != 0:
            msg = self.lib.sch_last_error(self.handle).decode(errors="replace")
            if rc == SCH_ERR_SOLVER:
                return rc
            raise RuntimeError(f"{name} failed (status {rc}): {msg}")
        return 0

    @property
    def launches(self) -> int:
        return int(self.lib.sch_launch_count(self.handle))


def ctx(device: int | None = None) -> Context:
    """The context of torch's current stream on ``device``."""
    if device is None:
        device = torch.cuda.current_device()
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    c = _contexts.get(key)
    if c is None:
        with _lock:
            c = _contexts.get(key)
            if c is None:
                c = Context(device, key[1])
                _contexts[key] = c
    return c


def ptr(t: torch.Tensor | None):
    if t is None:
        return None
    return _c_ptr(t.data_ptr())


def launch_count() -> int:
    """Kernels launched by this process's contexts (bench accounting)."""
    return sum(c.launches for c in _contexts.values())
