"""Host-side logic of the drop-in package and the C-ABI boundary (CPU only).

No compute call needs a GPU here: the C-ABI library must load and export
every symbol include/lcsgrid_b200.h declares, and the Python mirror must keep
the reference's argument checks, short-circuits and exception messages.
"""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2309_09072_b200 as L
from paper_2309_09072_b200 import _backend, _lib, seqcore

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lcsgrid_b200.h")).read()
    return sorted(set(re.findall(r"\b(lcsg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), "python bindings out of sync with the header"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_and_no_fallback_on_cpu():
    lib = _lib.load()
    assert lib.lcsg_abi_version() == 100
    if lib.lcsg_device_count() == 0:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            L.lcs("abc", "abd")
        g = L.GridModel("ab", "abc")
        with pytest.raises(RuntimeError, match="no CUDA device"):
            L.build_cost_table(g, 1, 3)


def test_empty_short_circuit_needs_no_device():
    # solver.py:255-256: either input empty -> LcsResult(0, b"", (), ())
    assert L.lcs("", "abc") == L.LcsResult(0, b"", (), ())
    assert L.lcs(b"abc", b"") == L.LcsResult(0, b"", (), ())
    g = L.GridModel("", "")
    assert L.assemble_lcs(g, np.array([1], dtype=np.int32)) == L.LcsResult(0, b"", (), ())


def test_backend_env_aliases(monkeypatch):
    for name in ("cython", "python", "cuda"):
        monkeypatch.setenv("LCSGRID_BACKEND", name)
        assert _backend.default_backend() == "cuda"
    monkeypatch.setenv("LCSGRID_BACKEND", "numba")
    with pytest.raises(ValueError, match="LCSGRID_BACKEND='numba' not available"):
        _backend.resolve(None)


def test_type_and_backend_errors():
    with pytest.raises(TypeError, match="expected str or bytes, got int"):
        L.lcs(5, "abc")
    with pytest.raises(ValueError, match="unknown backend 'numba'"):
        L.lcs("abc", "abc", backend="numba")
    # the reference's own backend names are aliases of the CUDA path (drop-in)
    assert _backend.resolve("cython") == "cuda"
    assert _backend.resolve("python") == "cuda"
    # an empty input returns before the backend is resolved (solver.py:255-256)
    assert L.lcs("", "abc", backend="numba") == L.LcsResult(0, b"", (), ())
    assert _backend.resolve(None) == "cuda"
    assert _backend.resolve("auto") == "cuda"
    assert L.active_backend() == "cuda"
    assert L.have_extension()


def test_build_preconditions():
    g = L.GridModel("abc", "abcd")
    for top, bottom in ((0, 2), (2, 2), (1, 5)):
        with pytest.raises(AssertionError):
            L.build_cost_table(g, top, bottom)


def test_seqcore_types():
    g = seqcore.GridModel("tcaggatt", "gatttatgcagg")
    assert (g.m, g.n, g.inf) == (8, 12, 14)
    assert g.row_arr.dtype == np.uint8 and g.col_arr.tobytes() == b"gatttatgcagg"
    assert L.match_positions("gatttatgcagg", "t").tolist() == [3, 4, 5, 7]
    assert L.match_positions("abc", "z").tolist() == []
    assert seqcore.diagonal_weight(seqcore.GridModel("tcaggatt", "gatttatgcagg"), 1, 3) == 1
    with pytest.raises(AssertionError):
        seqcore.diagonal_weight(g, 0, 1)
    r = L.LcsResult(5, b"tcagg", (3, 9, 10, 11, 12), (1, 2, 3, 4, 5))
    r.validate("gatttatgcagg", "tcaggatt")
    with pytest.raises(ValueError, match="not strictly increasing"):
        L.LcsResult(2, b"tt", (3, 3), (1, 2)).validate("gatttatgcagg", "tt")
    with pytest.raises(ValueError, match="length fields disagree"):
        L.LcsResult(1, b"", (), ()).validate("a", "a")


def test_dp_lcs_matches_reference_goldens(ref_lcs_pairs):
    import oracle as O
    for p in ref_lcs_pairs[:120]:
        a, b = bytes.fromhex(p["a"]), bytes.fromhex(p["b"])
        d = L.dp_lcs(a, b)
        assert d.length == p["length"]
        d.validate(a, b)
    # oracle.py:36-63 backtrack (diag > up > left): paper pair positions
    d = L.dp_lcs("gatttatgcagg", "tcaggatt")
    assert d.row_positions == (7, 9, 10, 11, 12)
    assert O.lcs("gatttatgcagg", "tcaggatt")[2] == (3, 9, 10, 11, 12)
