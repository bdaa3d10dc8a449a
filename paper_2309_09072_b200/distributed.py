"""Multi-GPU schedule of the Lu-Liu recursion.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on GPUs;
gloo works too, staged through host memory).  The reference builds its tree
depth-first on one CPU (solver.py:113-119); here P ranks split it:

* **bands** -- the P nodes at depth log2(P) of the reference tree (same
  ``mid=(top+bottom)//2`` split) are independent sub-problems: rank r builds
  band r's whole subtree with ``lcsg_build`` on that slab, with zero
  communication;
* **upper levels** -- every combine above the bands is sharded over start
  columns i: all ranks hold the full U and L tables, rank r computes rows
  [lo_r, hi_r) (contiguous ranges balanced by the per-row work proxy
  kmax_U[i] + 1) with ``lcsg_combine_rows``, then each owner broadcasts its
  reach/kmax row range so every rank ends with the full output table (traces
  stay with their owner: the walk needs one cell per upper node);
* **recovery** -- the walk over the upper nodes (solver.py:180-207) runs on
  every rank from the gathered tables and yields each band's (start column,
  weight); each band owner walks its own subtree (``lcsg_recover_from``) and
  the cross-vertex columns are gathered; every rank assembles the LcsResult.

The tree shape is the reference's, so every table -- and the final D_G, path,
subsequence and positions -- is bit-identical to the single-GPU solve and to
the reference.  The data-path collectives are broadcasts of finished row
ranges (an all-gather with uneven shards) plus one max all-reduce per combine.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Dict, Tuple, List, Optional

import numpy as np

from . import _lib
from .seqcore import GridModel, LcsResult, as_bytes


@dataclass
class Node:
    """A node of the reference recursion tree (solver.py:113-119)."""

    top: int
    bottom: int
    depth: int
    upper: Optional["Node"] = None
    lower: Optional["Node"] = None
    band: int = -1  # band index (owner rank) for band nodes
    table: dict = field(default_factory=dict)

    @property
    def rows(self) -> int:
        return self.bottom - self.top


def build_plan(m: int, P: int):
    """Reference tree cut at depth log2(P): (root, bands, upper nodes bottom-up).

    P is reduced to the largest power of two whose depth still has no leaves
    (every band must be a slab of >= 2 rows so that it is a combine)."""
    assert m >= 1 and P >= 1
    d = 0
    while (1 << (d + 1)) <= P and (m >> (d + 1)) >= 2:
        d += 1

    def mk(top, bottom, depth):
        nd = Node(top, bottom, depth)
        if depth < d:
            mid = (top + bottom) // 2
            nd.upper = mk(top, mid, depth + 1)
            nd.lower = mk(mid, bottom, depth + 1)
        return nd

    root = mk(1, m + 1, 0)
    bands: List[Node] = []
    upper: List[Node] = []

    def walk(nd):
        if nd.depth == d:
            nd.band = len(bands)
            bands.append(nd)
            return
        walk(nd.upper)
        walk(nd.lower)
        upper.append(nd)  # post-order == bottom-up, children first

    walk(root)
    return root, bands, upper


def split_rows(weights: np.ndarray, P: int):
    """Contiguous [lo, hi) row ranges with near-equal total weight (identical
    on every rank: a pure function of the gathered kmax row)."""
    n1 = len(weights)
    cum = np.concatenate([[0], np.cumsum(weights.astype(np.int64))])
    total = cum[-1]
    cuts = [0]
    for r in range(1, P):
        cuts.append(int(np.searchsorted(cum, total * r / P, side="left")))
    cuts.append(n1)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n1))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(P)]


class CudaBackend:
    """Device operations of the sharded schedule through the C-ABI."""

    def __init__(self, device: int):
        import torch

        self.torch = torch
        self.device = device
        self.dev = torch.device("cuda", device)
        self.lib = _lib.load()
        self.handles = []

    def stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.dev).cuda_stream)

    def empty(self, shape, dtype="int32"):
        return self.torch.empty(shape, dtype=getattr(self.torch, dtype), device=self.dev)

    def build_band(self, rows: bytes, cols: bytes, top: int, bottom: int, with_trace: bool):
        t = self.torch
        r = np.frombuffer(rows, dtype=np.uint8)
        c = np.frombuffer(cols, dtype=np.uint8) if len(cols) else np.zeros(1, np.uint8)
        h = ctypes.c_void_p()
        flags = _lib.LCSG_WITH_TRACE if with_trace else 0
        _lib.check(self.lib.lcsg_build(r.ctypes.data, len(r), c.ctypes.data, len(cols), top, bottom,
                                       flags, self.device, self.stream(), ctypes.byref(h)),
                   "band build")
        self.handles.append(h)
        root = self.lib.lcsg_root(h)
        info = (ctypes.c_int32 * 8)()
        _lib.check(self.lib.lcsg_node_info(h, root, info))
        n1, w1 = int(info[6]) + 1, int(info[2])
        p = ctypes.c_void_p()
        _lib.check(self.lib.lcsg_node_reach_device(h, root, ctypes.byref(p)))
        reach = self.empty((n1, w1))
        kmax_h = np.empty(n1, dtype=np.int32)
        _lib.check(self.lib.lcsg_node_kmax(h, root, kmax_h.ctypes.data))
        ws = ctypes.c_int32()
        _lib.check(self.lib.lcsg_node_wstar(h, root, ctypes.byref(ws)))

        class _Iface:
            __cuda_array_interface__ = {"shape": (n1, w1), "typestr": "<i4",
                                        "data": (int(p.value), False), "version": 3,
                                        "strides": None}

        reach.copy_(t.as_tensor(_Iface(), device=self.dev))
        return h, reach, t.from_numpy(kmax_h).to(self.dev), int(ws.value)

    def combine_rows(self, U, L, out, lo, hi, inf):
        _lib.check(self.lib.lcsg_combine_rows(
            U["reach"].data_ptr(), U["reach"].shape[1], U["kmax"].data_ptr(),
            L["reach"].data_ptr(), L["reach"].shape[1], L["kmax"].data_ptr(), int(L["wstar"]),
            out["reach"].data_ptr(), out["trace"].data_ptr(), out["kmax"].data_ptr(),
            out["wstar_dev"].data_ptr(), out["reach"].shape[1], inf, U["reach"].shape[0], lo, hi,
            self.stream()), "combine_rows")

    def recover_band(self, h, i_start: int, j: int, m_band: int):
        cols = np.empty(m_band + 1, dtype=np.int32)
        _lib.check(self.lib.lcsg_recover_from(h, int(i_start), int(j), cols.ctypes.data),
                   "band recovery")
        return cols

    def synchronize(self):
        self.torch.cuda.synchronize(self.dev)

    def assemble(self, g, path):
        from . import solver

        return solver.assemble_lcs(g, path, device=self.device)

    def free(self):
        for h in self.handles:
            self.lib.lcsg_free(h)
        self.handles = []


def _bcast(dist, group, t, src):
    """Broadcast a (possibly CUDA) tensor; gloo is staged through host memory."""
    if t.numel() == 0:
        return
    if t.is_cuda and dist.get_backend(group) == "gloo":
        tmp = t.cpu()
        dist.broadcast(tmp, src=src, group=group)
        t.copy_(tmp)
    else:
        dist.broadcast(t, src=src, group=group)


def _bcast_finite_rows(dist, group, table, kmax_rows, src, inf):
    """Broadcast rows of a reach table by their finite prefixes only.

    Row i holds finite values in columns 0..kmax[i] and INF beyond, so only
    those prefixes travel (about a third of a sigma=26 top-level table,
    SURVEY.md 8(e)); every rank already has ``kmax_rows``, so payload sizes
    need no exchange.  Receivers rebuild the rows with INF fill."""
    import torch

    if table.numel() == 0:
        return
    cols = torch.arange(table.shape[1], device=table.device, dtype=kmax_rows.dtype)
    mask = cols[None, :] <= kmax_rows[:, None]
    me = dist.get_rank()  # global rank: src is a global rank (subgroups too)
    if me == src:
        payload = table[mask]
    else:
        payload = torch.empty(int(mask.sum().item()), dtype=table.dtype, device=table.device)
    _bcast(dist, group, payload, src)
    if me != src:
        table.fill_(inf)
        table[mask] = payload


def _allreduce_max(dist, group, t):
    from torch.distributed import ReduceOp

    if t.is_cuda and dist.get_backend(group) == "gloo":
        tmp = t.cpu()
        dist.all_reduce(tmp, op=ReduceOp.MAX, group=group)
        t.copy_(tmp)
    else:
        dist.all_reduce(t, op=ReduceOp.MAX, group=group)


_SUBGROUPS: Dict[Tuple[int, Tuple[int, ...]], object] = {}


def _subgroup(dist, parent, ranks: Tuple[int, ...]):
    """Process group of a subtree's (global) ranks, created once per parent
    group and rank set: every rank asks for the same sets in the same order,
    so creation stays collective while repeated solves reuse communicators."""
    key = (id(parent), ranks)
    g = _SUBGROUPS.get(key)
    if g is None:
        g = dist.new_group(list(ranks))
        _SUBGROUPS[key] = g
    return g


def _rank_sets(root: Node, P: int) -> Dict[int, Tuple[int, ...]]:
    """Ranks that compute each node: a band its owner (band % P), an upper
    node the union of its children's ranks (the ranks of its subtree)."""
    rs: Dict[int, Tuple[int, ...]] = {}

    def f(nd):
        if nd.band >= 0:
            key = (nd.band % P,)
        else:
            key = tuple(sorted(set(f(nd.upper)) | set(f(nd.lower))))
        rs[id(nd)] = key
        return key

    f(root)
    return rs


def _replicate(dist, G, rank, ch: Node, ch_ranks, backend, n, inf):
    """Make child table ``ch`` (reach, kmax, wstar) complete on every rank of
    the parent's group ``G``: a band from its owner, an upper node from the
    owners of its row ranges (spans first, so that every member knows them);
    rows travel as finite prefixes."""
    import torch

    n1 = n + 1
    w1 = min(ch.rows, n) + 1
    if ch.band >= 0:
        spans = [(ch_ranks[0], 0, n1)]  # a band's rank set is its owner
    else:
        meta = backend.empty((3 * len(ch_ranks),))
        if ch.table is not None and "spans" in ch.table:
            meta.copy_(torch.tensor([v for sp in ch.table["spans"] for v in sp], dtype=meta.dtype))
        _bcast(dist, G, meta, ch_ranks[0])
        mh = meta.cpu().tolist()
        spans = [tuple(int(v) for v in mh[3 * t: 3 * t + 3]) for t in range(len(ch_ranks))]
    if ch.table is None:
        ch.table = {"handle": None}
    T = ch.table
    if "reach" not in T or T["reach"] is None:
        T["reach"] = backend.empty((n1, w1))
        T["kmax"] = backend.empty((n1,))
    # every member takes part (each child is replicated once, for its parent);
    # the owners of row ranges send, the others receive
    for owner, lo, hi in spans:
        _bcast(dist, G, T["kmax"][lo:hi], owner)
        _bcast_finite_rows(dist, G, T["reach"][lo:hi], T["kmax"][lo:hi], owner, inf)
    ws = torch.tensor([int(T.get("wstar", 0))], dtype=torch.int32, device=T["reach"].device)
    _bcast(dist, G, ws, spans[0][0])
    T["wstar"] = int(ws.item())
    T["reach_full"] = True
    T["spans"] = spans


def solve_sharded(rows: bytes, cols: bytes, dist, group=None, backend=None, with_trace=True):
    """Sharded build of the full-grid tree: returns (root, bands, upper, ctx).

    Bands are built by their owners with no communication.  Each upper
    combine is computed by the ranks of its own subtree (pairs, quads, ...,
    all ranks at the root), sharded over start columns; before it, the two
    children tables are replicated within that subtree's process group only
    (finite row prefixes), so a rank receives its sibling subtrees' tables,
    not every table of the level.  Traces and the root's rows stay with
    their row owners (``table["spans"]`` = (rank, lo, hi))."""
    import torch

    rank, P = dist.get_rank(group), dist.get_world_size(group)
    m, n = len(rows), len(cols)
    n1, inf = n + 1, n + 2
    root, bands, upper = build_plan(m, P)
    rs = _rank_sets(root, P)
    glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    groups: Dict[Tuple[int, ...], object] = {}
    for nd in upper:  # collective: same order on every rank
        key = rs[id(nd)]
        if key not in groups:
            groups[key] = group if len(key) == P else _subgroup(dist, group, tuple(glob(r) for r in key))
    # 1. bands: independent subtrees, zero communication
    for b in bands:
        if b.band % P == rank:
            h, reach, kmax, ws = backend.build_band(rows, cols, b.top, b.bottom, with_trace)
            b.table = {"handle": h, "reach": reach, "kmax": kmax, "wstar": ws,
                       "reach_full": True, "handle_owner": rank}
        else:
            b.table = None
    backend.synchronize()
    # 2. upper combines, bottom-up, each within its subtree's group
    for nd in upper:
        key = rs[id(nd)]
        if rank not in key:
            nd.table = None
            continue
        G = groups[key]
        for ch in (nd.upper, nd.lower):
            _replicate(dist, G, rank, ch, [glob(r) for r in rs[id(ch)]], backend, n, inf)
        U, L = nd.upper.table, nd.lower.table
        w1 = min(nd.rows, n) + 1
        out = {"reach": backend.empty((n1, w1)), "trace": backend.empty((n1, w1)),
               "kmax": backend.empty((n1,)), "wstar_dev": backend.empty((1,))}
        out["wstar_dev"].zero_()
        weights = U["kmax"].cpu().numpy().astype(np.int64) + 1
        spans = split_rows(weights, len(key))
        lo, hi = spans[key.index(rank)]
        backend.combine_rows(U, L, out, lo, hi, inf)
        backend.synchronize()
        _allreduce_max(dist, G, out["wstar_dev"])
        out["wstar"] = int(out["wstar_dev"].item())
        out["spans"] = [(glob(key[t]), a, b) for t, (a, b) in enumerate(spans)]
        nd.table = out
    ctx = {"rs": rs, "groups": groups, "glob": glob, "group": group}
    return root, bands, upper, ctx


def recover_sharded(root: Node, bands: List[Node], m: int, dist, group=None, backend=None,
                    ctx=None):
    """Cross-vertex columns of the LCS path (solver.py:180-207), stitched from
    the upper-level walk and the band walks.  Each rank walks only the path
    towards its own band: at a node, the owner of the trace row broadcasts
    (k, x) within the node's group; then every member follows the child
    whose subtree holds it."""
    import torch

    rank, P = dist.get_rank(group), dist.get_world_size(group)
    rs, groups, glob = ctx["rs"], ctx["groups"], ctx["glob"]
    grank = glob(rank)
    R = root.table
    # row 0 of the root (LCS length, path end) lives on the first rank of the
    # root's rank set (the first span is never empty); ranks outside the plan
    # (more ranks than bands) hold nothing and only receive
    r0 = glob(rs[id(root)][0])
    head = backend.empty((1,))
    if R is not None and grank == r0:
        head.copy_(R["kmax"][0:1])
    _bcast(dist, group, head, r0)
    length = int(head.item())
    start = {}  # band -> (i, j)

    def owner_of(nd, row):
        return next(r for r, a, b in nd.table["spans"] if a <= row < b)

    def walk(nd, i, jj):
        if nd.band >= 0:
            start[nd.band] = (i, jj)
            return
        G = groups[rs[id(nd)]]
        owner = owner_of(nd, i - 1)
        dev = nd.table["reach"].device
        kx = torch.zeros(2, dtype=torch.int32, device=dev)
        if grank == owner:
            k = int(nd.table["trace"][i - 1, jj].item())
            kx[0] = k
            kx[1] = int(nd.upper.table["reach"][i - 1, k].item())
        _bcast(dist, G, kx, owner)
        k, x = int(kx[0].item()), int(kx[1].item())
        if rank in rs[id(nd.upper)]:
            walk(nd.upper, i, k)
        if rank in rs[id(nd.lower)]:
            walk(nd.lower, x, jj - k)

    if rank in rs[id(root)]:
        walk(root, 1, length)
    cols = np.zeros(m + 1, dtype=np.int32)
    pieces = []
    for b in bands:
        if b.band % P == rank:
            i, jj = start[b.band]
            pieces.append((b.top, backend.recover_band(b.table["handle"], i, jj, b.rows)))
    gathered = [None] * P
    dist.all_gather_object(gathered, pieces, group=group)
    for plist in gathered:
        for top, seg in plist:
            cols[top - 1: top - 1 + len(seg)] = seg
    # the path's end column: root cell (start column 1, weight length), held by
    # the owner of row 0 (root rows are not replicated)
    end_owner = r0
    end = backend.empty((1,))
    if R is not None and grank == r0:
        end.copy_(R["reach"][0, length].reshape(1))
    _bcast(dist, group, end, end_owner)
    cols[m] = int(end.item())
    return length, cols


def lcs_sharded(a, b, *, group=None, device=None, low_memory=False, backend=None) -> LcsResult:
    """``lcs(a, b)`` (solver.py:237-273) across the ranks of ``group``; every
    rank returns the same LcsResult, bit-identical to the single-GPU solve."""
    import torch.distributed as dist

    aa, bb = as_bytes(a), as_bytes(b)
    if len(aa) == 0 or len(bb) == 0:
        return LcsResult(0, b"", (), ())
    swapped = len(aa) > len(bb)
    rows, cols = (bb, aa) if swapped else (aa, bb)
    own = backend is None
    if own:
        backend = CudaBackend(0 if device is None else int(device))
    try:
        root, bands, upper, ctx = solve_sharded(rows, cols, dist, group, backend,
                                                with_trace=not low_memory)
        length, path = recover_sharded(root, bands, len(rows), dist, group, backend, ctx)
    finally:
        if own:
            backend.free()
    r = backend.assemble(GridModel(rows, cols), path)
    if swapped:
        r = LcsResult(r.length, r.subsequence, r.col_positions, r.row_positions)
    return r
