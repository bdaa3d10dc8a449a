"""ctypes wrapper of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product package (paper_2309_09072_b200) never does.  It exposes
the CPU restatement in lcsgrid_oracle.c (which cites the reference
file:line for every function) with numpy in/out, mirroring the reference's
own Python signatures where one exists.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblcsgrid_oracle.so")
_lib = None

_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class _Node(ctypes.Structure):
    _fields_ = [
        ("top_row", ctypes.c_int32), ("bottom_row", ctypes.c_int32),
        ("w1", ctypes.c_int32), ("wstar", ctypes.c_int32),
        ("upper", ctypes.c_int32), ("lower", ctypes.c_int32),
        ("reach", _i32p), ("trace", _i32p), ("kmax", _i32p),
    ]


def build_library() -> str:
    """Compile the oracle with its Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build_library()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_base_case_row.argtypes = [_u8p, ctypes.c_int32, ctypes.c_uint8, _i32p]
        L.orc_combine_level.argtypes = [
            _i32p, ctypes.c_int32, _i32p, _i32p, ctypes.c_int32, ctypes.c_int32,
            _i32p, _i32p, ctypes.c_int32, ctypes.c_int, ctypes.c_int32,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
            ctypes.POINTER(ctypes.c_uint64)]
        L.orc_build.argtypes = [_u8p, ctypes.c_int32, _u8p, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_int, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_void_p)]
        L.orc_free.argtypes = [ctypes.c_void_p]
        L.orc_num_nodes.argtypes = [ctypes.c_void_p]
        L.orc_num_nodes.restype = ctypes.c_int32
        L.orc_root.argtypes = [ctypes.c_void_p]
        L.orc_root.restype = ctypes.c_int32
        L.orc_node_at.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.orc_node_at.restype = ctypes.POINTER(_Node)
        L.orc_counters.argtypes = [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_uint64)] * 4
        L.orc_recover.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i32p]
        L.orc_assemble.argtypes = [_u8p, ctypes.c_int32, _u8p, ctypes.c_int32, _i32p, _u8p,
                                   _i32p, _i32p]
        L.orc_assemble.restype = ctypes.c_int32
        L.orc_lcs.argtypes = [_u8p, ctypes.c_int32, _u8p, ctypes.c_int32, ctypes.c_int,
                              ctypes.c_int, _u8p, _i32p, _i32p]
        L.orc_lcs.restype = ctypes.c_int32
        _lib = L
    return _lib


def _u8(buf) -> np.ndarray:
    if isinstance(buf, str):
        buf = buf.encode("latin-1")
    return np.ascontiguousarray(np.frombuffer(bytes(buf), dtype=np.uint8))


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def inf_value(n: int) -> int:
    return n + 2


def base_case_row(cols, sym: int) -> np.ndarray:
    """breakout.py:37-55."""
    c = _u8(cols)
    out = np.empty(len(c), dtype=np.int32)
    if len(c):
        lib().orc_base_case_row(_p(c, _u8p), len(c), int(sym), _p(out, _i32p))
    return out


def combine_level(upper_reach, upper_kmax, lower_reach, lower_wstar, out_w1, inf,
                  with_trace=True, i_lo=0, i_hi=None, threads=1):
    """_kernel.pyx:63-82 on fresh output arrays; returns (reach, trace, ncell)."""
    U = np.ascontiguousarray(upper_reach, dtype=np.int32)
    K = np.ascontiguousarray(upper_kmax, dtype=np.int32)
    L = np.ascontiguousarray(lower_reach, dtype=np.int32)
    n1 = U.shape[0]
    if i_hi is None:
        i_hi = n1
    reach = np.zeros((n1, out_w1), dtype=np.int32)
    trace = np.zeros((n1, out_w1), dtype=np.int32)
    cnt = ctypes.c_uint64(0)
    lib().orc_combine_level(_p(U, _i32p), U.shape[1], _p(K, _i32p), _p(L, _i32p), L.shape[1],
                            int(lower_wstar), _p(reach, _i32p), _p(trace, _i32p), out_w1,
                            int(bool(with_trace)), int(inf), int(i_lo), int(i_hi), int(threads),
                            ctypes.byref(cnt), None)
    return reach, trace, int(cnt.value)


@dataclass
class OracleNode:
    top_row: int
    bottom_row: int
    reach: np.ndarray
    trace: Optional[np.ndarray]
    kmax: np.ndarray
    wstar: int
    upper: int
    lower: int


class OracleTree:
    """The whole reference recursion tree (solver.py:113-119), node order =
    reference creation order (post-order: upper subtree, lower subtree, self)."""

    def __init__(self, rows, cols, top_row=1, bottom_row=None, with_trace=True, threads=1,
                 count=False):
        r, c = _u8(rows), _u8(cols)
        self.m, self.n = len(r), len(c)
        self.inf = inf_value(self.n)
        if bottom_row is None:
            bottom_row = self.m + 1
        h = ctypes.c_void_p()
        rc = lib().orc_build(_p(r, _u8p) if len(r) else None, self.m,
                             _p(c, _u8p) if len(c) else None, self.n, int(top_row),
                             int(bottom_row), int(bool(with_trace)) | (2 if count else 0),
                             int(threads), ctypes.byref(h))
        if rc != 0:
            raise AssertionError("1 <= top_row < bottom_row <= m + 1")
        self._h = h
        self._rows, self._cols = r, c

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.orc_free(h)
            self._h = None

    @property
    def root(self) -> int:
        return lib().orc_root(self._h)

    def __len__(self) -> int:
        return lib().orc_num_nodes(self._h)

    def node(self, idx: int) -> OracleNode:
        nd = lib().orc_node_at(self._h, idx).contents
        n1 = self.n + 1
        reach = np.ctypeslib.as_array(nd.reach, shape=(n1, nd.w1)).copy()
        trace = (np.ctypeslib.as_array(nd.trace, shape=(n1, nd.w1)).copy()
                 if bool(nd.trace) else None)
        kmax = np.ctypeslib.as_array(nd.kmax, shape=(n1,)).copy()
        return OracleNode(nd.top_row, nd.bottom_row, reach, trace, kmax, nd.wstar,
                          nd.upper, nd.lower)

    def nodes(self) -> List[OracleNode]:
        return [self.node(i) for i in range(len(self))]

    def counters(self):
        """Reference work counts: Alg. 1 cell evaluations
        C, L gathers G, combine output cells OUT, combine input cells IN.
        C and G are only counted when the tree was built with count=True."""
        a, g, b, c = (ctypes.c_uint64() for _ in range(4))
        lib().orc_counters(self._h, ctypes.byref(a), ctypes.byref(g), ctypes.byref(b),
                           ctypes.byref(c))
        return dict(C=int(a.value), G=int(g.value), OUT=int(b.value), IN=int(c.value))

    def recover(self, j: int) -> np.ndarray:
        """solver.py:180-207."""
        out = np.empty(self.m + 1, dtype=np.int32)
        rc = lib().orc_recover(self._h, int(j), _p(out, _i32p))
        if rc == -1:
            raise ValueError("recovery needs the full-grid table")
        if rc == -2:
            raise ValueError(f"no path of weight {j} exists")
        return out


def assemble(rows, cols, path):
    """solver.py:210-234 -> (length, subsequence, row_positions, col_positions)."""
    r, c = _u8(rows), _u8(cols)
    p = np.ascontiguousarray(path, dtype=np.int32)
    k = max(1, min(len(r), len(c)))
    sub = np.empty(k, dtype=np.uint8)
    rp = np.empty(k, dtype=np.int32)
    cp = np.empty(k, dtype=np.int32)
    n = lib().orc_assemble(_p(r, _u8p) if len(r) else None, len(r),
                           _p(c, _u8p) if len(c) else None, len(c), _p(p, _i32p),
                           _p(sub, _u8p), _p(rp, _i32p), _p(cp, _i32p))
    return n, sub[:n].tobytes(), tuple(int(x) for x in rp[:n]), tuple(int(x) for x in cp[:n])


def lcs(a, b, low_memory=False, threads=1):
    """solver.py:237-273 -> (length, subsequence, positions_in_a, positions_in_b)."""
    x, y = _u8(a), _u8(b)
    k = max(1, min(len(x), len(y)))
    sub = np.empty(k, dtype=np.uint8)
    pa = np.empty(k, dtype=np.int32)
    pb = np.empty(k, dtype=np.int32)
    n = lib().orc_lcs(_p(x, _u8p) if len(x) else None, len(x),
                      _p(y, _u8p) if len(y) else None, len(y), int(bool(low_memory)),
                      int(threads), _p(sub, _u8p), _p(pa, _i32p), _p(pb, _i32p))
    if n < 0:
        raise RuntimeError("oracle build failed")
    return n, sub[:n].tobytes(), tuple(int(v) for v in pa[:n]), tuple(int(v) for v in pb[:n])
