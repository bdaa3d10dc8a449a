"""Drop-in solver entry points of the reference (solver.py), on the GPU.

Same names, signatures, argument meanings and exception types as the
reference package's ``lcsgrid.solver`` (file:line cited per function); each
call goes through the C-ABI library to hand-written sm_100a kernels.  The
``threads`` argument is accepted and ignored (the CUDA grid replaces the CPU
pool); ``backend`` accepts only None / "auto" / "cuda".
"""

from __future__ import annotations

import ctypes
from concurrent.futures import ThreadPoolExecutor
from typing import Optional

import numpy as np

from . import _backend, _lib
from .seqcore import BreakoutRow, GridModel, LcsResult, SequenceLike, as_bytes


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Tree:
    """Owner of one device-resident recursion tree (an lcsg_handle)."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                _lib.load().lcsg_free(h)
            except Exception:  # interpreter shutdown
                pass
            self.handle = None


class CostTable:
    """Reach table of one slab (reference solver.py:32-62), resident in HBM.

    ``reach`` / ``trace`` / ``kmax`` are copied to host numpy arrays on first
    access (byte-identical to the reference's arrays); ``reach_device`` is a
    zero-copy torch view of the device buffer.  ``upper`` / ``lower`` expose
    the child slabs of the same device tree.
    """

    def __init__(self, tree: _Tree, node: int):
        self._tree = tree
        self._node = node
        info = (ctypes.c_int32 * 8)()
        _lib.check(_lib.load().lcsg_node_info(tree.handle, node, info), "node_info")
        (self.top_row, self.bottom_row, self._w1, self._upper, self._lower, self._has_trace,
         self.n, self.inf) = (int(v) for v in info)
        self._cache = {}

    # -- reference fields ---------------------------------------------------
    @property
    def reach(self) -> np.ndarray:
        if "reach" not in self._cache:
            out = np.empty((self.n + 1, self._w1), dtype=np.intc)
            _lib.check(_lib.load().lcsg_node_reach(self._tree.handle, self._node, _ptr(out)))
            self._cache["reach"] = out
        return self._cache["reach"]

    @property
    def trace(self) -> Optional[np.ndarray]:
        if not self._has_trace:
            return None
        if "trace" not in self._cache:
            out = np.empty((self.n + 1, self._w1), dtype=np.intc)
            _lib.check(_lib.load().lcsg_node_trace(self._tree.handle, self._node, _ptr(out)))
            self._cache["trace"] = out
        return self._cache["trace"]

    @property
    def kmax(self) -> np.ndarray:
        if "kmax" not in self._cache:
            out = np.empty(self.n + 1, dtype=np.intc)
            _lib.check(_lib.load().lcsg_node_kmax(self._tree.handle, self._node, _ptr(out)))
            self._cache["kmax"] = out
        return self._cache["kmax"]

    @property
    def wstar(self) -> int:
        v = ctypes.c_int32()
        _lib.check(_lib.load().lcsg_node_wstar(self._tree.handle, self._node, ctypes.byref(v)))
        return int(v.value)

    @property
    def upper(self) -> Optional["CostTable"]:
        return CostTable(self._tree, self._upper) if self._upper >= 0 else None

    @property
    def lower(self) -> Optional["CostTable"]:
        return CostTable(self._tree, self._lower) if self._lower >= 0 else None

    @property
    def max_weight(self) -> int:
        return self._w1 - 1

    def row(self, i: int) -> BreakoutRow:
        """Reach vector of start column i (1-based, up to n + 1)."""
        assert 1 <= i <= self.n + 1
        return BreakoutRow(start=i, reach=self.reach[i - 1])

    # -- device access --------------------------------------------------------
    @property
    def reach_device(self):
        """Zero-copy torch.int32 CUDA view (n+1, w1) of the device table."""
        import torch

        p = ctypes.c_void_p()
        _lib.check(_lib.load().lcsg_node_reach_device(self._tree.handle, self._node,
                                                      ctypes.byref(p)))
        shape = (self.n + 1, self._w1)

        class _Iface:
            __cuda_array_interface__ = {
                "shape": shape, "typestr": "<i4", "data": (int(p.value or 0), False),
                "version": 3, "strides": None,
            }

        t = torch.as_tensor(_Iface(), device=f"cuda:{self._tree.device}")
        t._lcsg_owner = self._tree  # keep the device tree alive with the view
        return t


def _device(device) -> int:
    return 0 if device is None else int(device)


def build_cost_table(
    g: GridModel,
    top_row: int,
    bottom_row: int,
    *,
    threads: int = 1,
    backend=None,
    with_trace: bool = True,
    device=None,
) -> CostTable:
    """Reach table of the slab of vertex rows [top_row, bottom_row]
    (reference solver.py:122-139): the whole recursion runs on the GPU, one
    batched launch per tree height."""
    assert 1 <= top_row < bottom_row <= g.m + 1
    _backend.resolve(backend)
    L = _lib.load()
    rows = np.frombuffer(g.row_seq, dtype=np.uint8) if g.m else np.zeros(1, np.uint8)
    cols = np.frombuffer(g.col_seq, dtype=np.uint8) if g.n else np.zeros(1, np.uint8)
    h = ctypes.c_void_p()
    flags = _lib.LCSG_WITH_TRACE if with_trace else 0
    dev = _device(device)
    rc = L.lcsg_build(_ptr(rows), g.m, _ptr(cols), g.n, int(top_row), int(bottom_row), flags, dev,
                      None, ctypes.byref(h))
    _lib.check(rc, "build_cost_table")
    tree = _Tree(h, dev)
    _lib.check(L.lcsg_sync(h), "build_cost_table")
    return CostTable(tree, int(L.lcsg_root(h)))


def combine_row(upper_row: BreakoutRow, lower: CostTable, max_weight: int):
    """Merge one start column's reach vector with the slab below it
    (reference solver.py:142-157), through the device combine kernel."""
    import torch

    inf = lower.inf
    urow = np.ascontiguousarray(upper_row.reach, dtype=np.intc)
    kmax_i = int((urow < inf).sum()) - 1
    dev = lower._tree.device
    U = torch.from_numpy(urow.reshape(1, -1)).to(f"cuda:{dev}")
    K = torch.tensor([kmax_i], dtype=torch.int32, device=f"cuda:{dev}")
    Ld = lower.reach_device
    reach = torch.empty((1, max_weight + 1), dtype=torch.int32, device=f"cuda:{dev}")
    trace = torch.empty_like(reach)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = _lib.load().lcsg_combine_level(
        U.data_ptr(), U.shape[1], K.data_ptr(), Ld.data_ptr(), Ld.shape[1], lower.wstar,
        reach.data_ptr(), trace.data_ptr(), max_weight + 1, 1, inf, 1, 0, 1, stream)
    _lib.check(rc, "combine_row")
    return (BreakoutRow(start=upper_row.start, reach=reach.cpu().numpy()[0].astype(np.intc)),
            trace.cpu().numpy()[0].astype(np.intc))


def lcs_length(table: CostTable) -> int:
    """Largest weight reachable from start column 1 (reference solver.py:160-162)."""
    if table._node != _lib.load().lcsg_root(table._tree.handle):
        return int(table.kmax[0])
    v = ctypes.c_int32()
    _lib.check(_lib.load().lcsg_length(table._tree.handle, ctypes.byref(v)), "lcs_length")
    return int(v.value)


def recover_cross_vertices(g: GridModel, table: CostTable, j: int) -> np.ndarray:
    """Leftmost path column on every grid row for the weight-j path from the
    top-left start (reference solver.py:180-207), walked on the device."""
    m = g.m
    if not (table.top_row == 1 and table.bottom_row == m + 1):
        raise ValueError("recovery needs the full-grid table")
    length = lcs_length(table)
    if j > length:
        raise ValueError(f"no path of weight {j} exists (max {length})")
    cols = np.empty(m + 1, dtype=np.intc)
    _lib.check(_lib.load().lcsg_recover(table._tree.handle, int(j), _ptr(cols)),
               "recover_cross_vertices")
    return cols


def assemble_lcs(g: GridModel, path_cols: np.ndarray, *, device=None) -> LcsResult:
    """Read the subsequence off a cross-vertex path (reference
    solver.py:210-234): mark + scan + compact kernel on the device."""
    m, n = g.m, g.n
    if m == 0 or n == 0:
        return LcsResult(0, b"", (), ())
    path = np.ascontiguousarray(path_cols, dtype=np.int32)
    k = min(m, n)
    length = ctypes.c_int32()
    sub = np.empty(k, dtype=np.uint8)
    rp = np.empty(k, dtype=np.int32)
    cp = np.empty(k, dtype=np.int32)
    rows = np.frombuffer(g.row_seq, dtype=np.uint8)
    cols = np.frombuffer(g.col_seq, dtype=np.uint8)
    rc = _lib.load().lcsg_assemble(_ptr(rows), m, _ptr(cols), n, _ptr(path), _device(device),
                                   ctypes.byref(length), _ptr(sub), _ptr(rp), _ptr(cp))
    _lib.check(rc, "assemble_lcs")
    L = int(length.value)
    return LcsResult(length=L, subsequence=sub[:L].tobytes(),
                     row_positions=tuple(rp[:L].tolist()),
                     col_positions=tuple(cp[:L].tolist()))


def lcs(
    a: SequenceLike,
    b: SequenceLike,
    *,
    threads: int = 1,
    backend=None,
    low_memory: bool = False,
    device=None,
    stream=None,
) -> LcsResult:
    """One longest common subsequence of ``a`` and ``b`` (reference
    solver.py:237-273).  The shorter input indexes grid rows (ties keep ``a``
    as rows); output is identical to the reference for any input.
    ``low_memory`` drops stored traces and recomputes split weights on the
    recovery walk (solver.py:165-177), on the device.  Extensions beyond the
    reference signature (keyword-only): ``device`` (CUDA ordinal) and
    ``stream`` (a cudaStream_t handle as int, e.g. torch's current stream)."""
    aa = as_bytes(a)
    bb = as_bytes(b)
    if len(aa) == 0 or len(bb) == 0:  # before any backend resolution (solver.py:255-256)
        return LcsResult(0, b"", (), ())
    _backend.resolve(backend)
    k = min(len(aa), len(bb))
    x = np.frombuffer(aa, dtype=np.uint8)
    y = np.frombuffer(bb, dtype=np.uint8)
    length = ctypes.c_int32()
    sub = np.empty(k, dtype=np.uint8)
    pa = np.empty(k, dtype=np.int32)
    pb = np.empty(k, dtype=np.int32)
    flags = 0 if low_memory else _lib.LCSG_WITH_TRACE
    rc = _lib.load().lcsg_lcs(_ptr(x), len(aa), _ptr(y), len(bb), flags, _device(device), stream,
                              ctypes.byref(length), _ptr(sub), _ptr(pa), _ptr(pb))
    _lib.check(rc, "lcs")
    L = int(length.value)
    return LcsResult(length=L, subsequence=sub[:L].tobytes(),
                     row_positions=tuple(pa[:L].tolist()),
                     col_positions=tuple(pb[:L].tolist()))


def reserve(nbytes: int, *, device=None) -> None:
    """Map ``nbytes`` of HBM into the library's memory pool now (a serving
    process calls this at start-up, so its first large solve does not pay for
    the pool growth).  No reference counterpart."""
    _lib.check(_lib.load().lcsg_reserve(_device(device), int(nbytes)), "reserve")


def trim(*, device=None) -> None:
    """Return the pool's unused HBM (and the per-shape graph cache's arenas)
    to the driver.  No reference counterpart."""
    _lib.check(_lib.load().lcsg_trim(_device(device)), "trim")


def sweep_errors(*, device=None, reset: bool = False) -> int:
    """Consistency violations counted by the row-sweep kernels on ``device``
    since the last reset (0 unless a structural invariant failed; tests and
    ``bench.py`` assert it).  No reference counterpart."""
    import ctypes

    cnt = ctypes.c_int32(0)
    _lib.check(_lib.load().lcsg_sweep_errors(_device(device), ctypes.byref(cnt), int(reset)),
               "sweep_errors")
    return int(cnt.value)


def sweep_paths(*, device=None, reset: bool = False):
    """(blocks redone by the generic sweep kernel after a register-kernel flag,
    blocks swept with the row state in the output rows) since the last reset.
    Diagnostic; no reference counterpart."""
    import ctypes

    a, b = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(_lib.load().lcsg_sweep_paths(_device(device), ctypes.byref(a), ctypes.byref(b),
                                            int(reset)), "sweep_paths")
    return int(a.value), int(b.value)


# cells (m * n * pairs) per batched launch: bounds the batch's HBM arena
# (~125 B per cell-equivalent with traces at cfg5-like shapes)
_BATCH_CELLS = 1 << 28


def lcs_batch(
    a_list,
    b_list,
    *,
    threads: int = 1,
    backend=None,
    low_memory: bool = False,
    device=None,
    stream=None,
) -> list:
    """``[lcs(a, b) for a, b in zip(a_list, b_list)]`` for pairs of EQUAL
    shape (every a the same length, every b the same length), solved as ONE
    batch on the GPU: the recursion trees of all pairs are built together,
    one launch per tree height for the whole batch (
    reference row-range contract _kernel.pyx:63-82), then one walk and one
    assembly.  Results are identical to the per-pair calls."""
    A = [as_bytes(x) for x in a_list]
    Bs = [as_bytes(x) for x in b_list]
    if len(A) != len(Bs):
        raise ValueError("a_list and b_list differ in length")
    if not A:
        return []
    la, lb = len(A[0]), len(Bs[0])
    if any(len(x) != la for x in A) or any(len(x) != lb for x in Bs):
        raise ValueError("lcs_batch needs pairs of equal shape")
    if la == 0 or lb == 0:  # solver.py:255-256
        return [LcsResult(0, b"", (), ()) for _ in A]
    _backend.resolve(backend)
    npairs = len(A)
    k = min(la, lb)
    aa = np.frombuffer(b"".join(A), dtype=np.uint8)
    bb = np.frombuffer(b"".join(Bs), dtype=np.uint8)
    lengths = np.empty(npairs, dtype=np.int32)
    sub = np.empty(npairs * k, dtype=np.uint8)
    pa = np.empty(npairs * k, dtype=np.int32)
    pb = np.empty(npairs * k, dtype=np.int32)
    flags = 0 if low_memory else _lib.LCSG_WITH_TRACE
    rc = _lib.load().lcsg_lcs_batch(_ptr(aa), la, _ptr(bb), lb, npairs, flags, _device(device),
                                    stream, _ptr(lengths), _ptr(sub), _ptr(pa), _ptr(pb))
    _lib.check(rc, "lcs_batch")
    out = []
    for p in range(npairs):
        L = int(lengths[p])
        o = p * k
        out.append(LcsResult(length=L, subsequence=sub[o:o + L].tobytes(),
                             row_positions=tuple(pa[o:o + L].tolist()),
                             col_positions=tuple(pb[o:o + L].tolist())))
    return out


def lcs_many(
    pairs,
    *,
    threads: int = 1,
    backend=None,
    low_memory: bool = False,
    device=None,
    concurrency: int = 8,
    batch: bool = True,
) -> list:
    """``[lcs(a, b) for a, b in pairs]`` with the GPU shared across pairs
    (many small pairs, e.g. the planted queries of
    cfg4).  Pairs of equal shape are solved together by :func:`lcs_batch`
    (one launch per tree height for the group, chunked to bound memory);
    the remaining pairs run as independent solves on separate CUDA streams
    from ``concurrency`` host worker threads (the C-ABI call releases the
    GIL).  Results are identical to the sequential calls, in order."""
    _backend.resolve(backend)
    items = [(as_bytes(a), as_bytes(b)) for a, b in pairs]
    out = [None] * len(items)
    single = []
    if batch:
        groups = {}
        for idx, (a, b) in enumerate(items):
            groups.setdefault((len(a), len(b)), []).append(idx)
        for (la, lb), idxs in groups.items():
            if len(idxs) < 2 or la == 0 or lb == 0:
                single.extend(idxs)
                continue
            per = max(1, _BATCH_CELLS // max(1, la * lb))
            for c0 in range(0, len(idxs), per):
                chunk = idxs[c0:c0 + per]
                if len(chunk) == 1:
                    single.extend(chunk)
                    continue
                res = lcs_batch([items[i][0] for i in chunk], [items[i][1] for i in chunk],
                                low_memory=low_memory, device=device)
                for i, r in zip(chunk, res):
                    out[i] = r
    else:
        single = list(range(len(items)))
    single.sort()

    def one(i):
        a, b = items[i]
        return lcs(a, b, threads=threads, low_memory=low_memory, device=device)

    if concurrency <= 1 or len(single) <= 1:
        for i in single:
            out[i] = one(i)
        return out
    with ThreadPoolExecutor(max_workers=min(concurrency, len(single))) as ex:
        for i, r in zip(single, ex.map(one, single)):
            out[i] = r
    return out
