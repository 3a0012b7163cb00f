"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/schwinger_sm100.h declares, and the ctypes table matches the
header one to one."""

import ctypes

import numpy as np
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "schwinger_sm100.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|unsigned long long)\s+(sch_\w+)\(",
                                 text, re.M)))


def test_library_exists_and_loads():
    from paper_1512_03812_b200 import _lib
    assert _lib.LIB_PATH.exists(), "build the library first (__graft_entry__.build())"
    lib = _lib.load()
    assert b"sm_100a" in lib.sch_build_info()


def test_every_header_symbol_is_exported():
    from paper_1512_03812_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s


def test_ctypes_table_matches_header():
    from paper_1512_03812_b200 import _lib
    assert sorted(_lib.exported_symbols()) == header_symbols()


def test_header_argument_counts_match_ctypes():
    """Each ctypes argtypes list has as many entries as the C prototype."""
    from paper_1512_03812_b200 import _lib
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    protos = dict(re.findall(r"(sch_\w+)\(([^)]*)\)\s*;", text))
    for name, argtypes in _lib._SIGNATURES.items():
        args = [a for a in protos[name].split(",") if a.strip() and a.strip() != "void"]
        assert len(args) == len(argtypes), name


def test_library_is_sm100a_only():
    import subprocess
    from paper_1512_03812_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_no_cuda_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1512_03812_b200 as sw
    from paper_1512_03812_b200._lib import NativeUnavailable
    with pytest.raises(NativeUnavailable):
        sw.WilsonDirac([[[0.0, 0.0], [0.0, 0.0]]] * 2, 0.1)


def test_package_does_not_import_oracle():
    """The product path never touches the CPU oracle (test infrastructure)."""
    pkg = ROOT / "paper_1512_03812_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, re.M), f
        assert "schwinger_oracle" not in src, f


def test_np_rng_state_layout_matches_host_view():
    """The device Philox record is NumPy's state in 88 B (host view in lattice.py)."""
    from paper_1512_03812_b200 import _lib, lattice
    assert int(_lib.load().sch_np_rng_state_bytes()) == lattice._NP_STATE_DTYPE.itemsize == 88
    raw = np.zeros(2 * 88, dtype=np.uint8)
    rec = lattice._np_state_records(raw)
    rec["ctr"][1] = [1, 2, 3, 4]
    rec["pos"][1] = 3
    assert raw[88:96].view("<u8")[0] == 1 and raw[88 + 80:88 + 84].view("<i4")[0] == 3
