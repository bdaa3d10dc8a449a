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


def _is_gloo(dist, group):
    return dist.get_backend(group) == "gloo"


def _bcast(dist, group, t, src):
    """Broadcast a (possibly CUDA) tensor; gloo is staged through host memory."""
    if t.numel() == 0:
        return
    if t.is_cuda and _is_gloo(dist, group):
        tmp = t.cpu()
        dist.broadcast(tmp, src=src, group=group)
        t.copy_(tmp)
    else:
        dist.broadcast(t, src=src, group=group)


def _all_gather(dist, group, out, inp):
    """all_gather_into_tensor (equal shards; gloo staged through host memory)."""
    if inp.is_cuda and _is_gloo(dist, group):
        tmp = out.cpu()
        dist.all_gather_into_tensor(tmp, inp.cpu(), group=group)
        out.copy_(tmp)
    else:
        dist.all_gather_into_tensor(out, inp, group=group)


def _all_reduce_max(dist, group, t):
    from torch.distributed import ReduceOp

    if t.is_cuda and _is_gloo(dist, group):
        tmp = t.cpu()
        dist.all_reduce(tmp, op=ReduceOp.MAX, group=group)
        t.copy_(tmp)
    else:
        dist.all_reduce(t, op=ReduceOp.MAX, group=group)


_SUBGROUPS: Dict[Tuple[int, Tuple[int, ...]], object] = {}


def _subgroup(dist, parent, ranks: Tuple[int, ...]):
    """Process group of a subtree's (global) ranks, created once per parent
    group and rank set and reused by later solves.  Only the members call
    ``new_group`` (local synchronisation), so a ``group=`` that is a proper
    subgroup of the world does not hang the ranks outside it."""
    key = (id(parent), ranks)
    g = _SUBGROUPS.get(key)
    if g is None:
        g = dist.new_group(list(ranks), use_local_synchronization=True)
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


def _finite_index(kmax_rows, lo: int, total: int):
    """(row, column) of every finite cell of rows lo.. of a reach table --
    row i holds finite values in columns 0..kmax[i] (solver.py:84,104) -- in
    row-major order: the device-side pack / unpack index of a finite-prefix
    transfer (a prefix sum of the row lengths; ``total`` is known on the host,
    so nothing waits on the device)."""
    import torch

    counts = kmax_rows.long() + 1
    dev = kmax_rows.device
    rows = torch.repeat_interleave(torch.arange(lo, lo + len(counts), device=dev), counts,
                                   output_size=total)
    starts = torch.cumsum(counts, 0) - counts
    cols = torch.arange(total, device=dev) - starts[rows - lo]
    return rows, cols


class CommStats:
    """Bytes this rank received through the schedule's collectives."""

    def __init__(self):
        self.received = 0
        self.collectives = 0

    def add(self, gathered_bytes: int, own_bytes: int):
        self.received += gathered_bytes - own_bytes
        self.collectives += 1


def _replicate_children(dist, G, grank, members, nd: Node, rs, glob, backend, n, inf, stats):
    """Make both children tables of upper node ``nd`` (reach, kmax, wstar)
    complete on every member of its group ``G``, with two collectives and
    one host synchronisation:

    1. one all-gather of a fixed-size record per member -- for each child the
       row span it computed (a band owner: all rows), its partial wstar and
       its kmax rows -- from which every member knows both children's spans,
       full kmax rows and wstar (one device-to-host copy);
    2. one all-gather of the reach rows as finite prefixes (kmax[i] + 1
       entries; receivers refill the INF tail -- about a third of a sigma=26
       top-level table), padded to the largest member's
       payload, packed and unpacked on the device (``_finite_index``)."""
    import torch

    n1 = n + 1
    kids = (nd.upper, nd.lower)
    M = len(members)
    rec = 4 + n1  # per child: lo, hi, wstar part, has-rows, then kmax (n1)
    mine = backend.empty((2 * rec,))
    mine.zero_()
    for c, ch in enumerate(kids):
        T = ch.table
        if T is not None and "my_span" in T:
            lo, hi = T["my_span"]
            head = torch.tensor([lo, hi, 0, 1], dtype=mine.dtype)
            mine[c * rec: c * rec + 4].copy_(head)
            mine[c * rec + 2: c * rec + 3].copy_(T["wstar_part"].reshape(1))
            mine[c * rec + 4 + lo: c * rec + 4 + hi].copy_(T["kmax"][lo:hi])
    gathered = backend.empty((M * 2 * rec,))
    _all_gather(dist, G, gathered, mine)
    stats.add(gathered.numel() * 4, mine.numel() * 4)
    gd = gathered.view(M, 2, rec)
    gh = gd.cpu().numpy()  # the schedule's one host synchronisation per combine
    for c, ch in enumerate(kids):
        w1 = min(ch.rows, n) + 1
        if ch.table is None:
            ch.table = {"handle": None}
        T = ch.table
        spans, kmax_dev, wstar = [], backend.empty((n1,)), 0
        for t in range(M):
            lo, hi, ws, has = (int(v) for v in gh[t, c, :4])
            if not has:
                continue
            spans.append((members[t], lo, hi))
            kmax_dev[lo:hi].copy_(gd[t, c, 4 + lo: 4 + hi])
            wstar = max(wstar, ws)
        spans.sort(key=lambda sp: sp[1])
        kmax_h = np.zeros(n1, dtype=np.int64)
        for r, lo, hi in spans:
            kmax_h[lo:hi] = gh[members.index(r), c, 4 + lo: 4 + hi]
        if "reach" not in T or T["reach"] is None:
            T["reach"] = backend.empty((n1, w1))
        T["kmax"] = kmax_dev
        T["kmax_host"] = kmax_h
        T["wstar"] = wstar
        T["spans"] = spans
    # 2. finite prefixes of the reach rows, packed per member
    sizes = np.zeros((M, 2), dtype=np.int64)
    for c, ch in enumerate(kids):
        kh = ch.table["kmax_host"]
        for r, lo, hi in ch.table["spans"]:
            sizes[members.index(r), c] = int(kh[lo:hi].sum()) + (hi - lo)
    pad = int(sizes.sum(1).max()) if M else 0
    me = members.index(grank)
    payload = backend.empty((max(pad, 1),))
    off = 0
    for c, ch in enumerate(kids):
        T = ch.table
        if "my_span" in T:
            lo, hi = T["my_span"]
            tot = int(sizes[me, c])
            if tot:
                rows, cols = _finite_index(T["kmax"][lo:hi], lo, tot)
                payload[off: off + tot].copy_(T["reach"][rows, cols])
            off += tot
    allp = backend.empty((M * max(pad, 1),))
    _all_gather(dist, G, allp, payload)
    stats.add(allp.numel() * 4, payload.numel() * 4)
    allp = allp.view(M, max(pad, 1))
    for c, ch in enumerate(kids):
        T = ch.table
        pieces = []
        for r, lo, hi in T["spans"]:
            t = members.index(r)
            o = int(sizes[t, :c].sum())
            pieces.append(allp[t, o: o + int(sizes[t, c])])
        flat = torch.cat(pieces) if pieces else allp.new_empty((0,))
        total = int(flat.numel())
        reach = T["reach"]
        reach.fill_(inf)
        if total:
            rows, cols = _finite_index(T["kmax"], 0, total)
            reach[rows, cols] = flat
        T["reach_full"] = True


def solve_sharded(rows: bytes, cols: bytes, dist, group=None, backend=None, with_trace=True,
                  stats: Optional[CommStats] = None):
    """Sharded build of the full-grid tree: returns (root, bands, upper, ctx).

    Bands are built by their owners with no communication.  Each upper
    combine is computed by the ranks of its own subtree (pairs, quads, ...,
    all ranks at the root), sharded over start columns; before it, the two
    children tables are replicated within that subtree's process group only
    (``_replicate_children``: two all-gathers, one host synchronisation), so
    a rank receives its sibling subtrees' tables, not every table of the
    level.  Traces and the root's rows stay with their row owners
    (``table["spans"]`` = (global rank, lo, hi)).  Nothing else waits on the
    device: the row split of a combine is a pure function of the gathered
    kmax rows, and partial wstar values travel in the next gather."""
    import torch

    stats = stats if stats is not None else CommStats()
    rank, P = dist.get_rank(group), dist.get_world_size(group)
    m, n = len(rows), len(cols)
    n1, inf = n + 1, n + 2
    root, bands, upper = build_plan(m, P)
    rs = _rank_sets(root, P)
    glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    grank = glob(rank)
    groups: Dict[Tuple[int, ...], object] = {}
    for nd in upper:  # members create their subtree's group (same order everywhere)
        key = rs[id(nd)]
        if key not in groups and rank in key:
            groups[key] = group if len(key) == P else _subgroup(dist, group, tuple(glob(r) for r in key))
    # 1. bands: independent subtrees, zero communication
    for b in bands:
        if b.band % P == rank:
            h, reach, kmax, ws = backend.build_band(rows, cols, b.top, b.bottom, with_trace)
            b.table = {"handle": h, "reach": reach, "kmax": kmax, "wstar": ws,
                       "wstar_part": torch.tensor([ws], dtype=torch.int32, device=reach.device),
                       "my_span": (0, n1), "reach_full": True, "handle_owner": rank}
        else:
            b.table = None
    # 2. upper combines, bottom-up, each within its subtree's group
    for nd in upper:
        key = rs[id(nd)]
        if rank not in key:
            nd.table = None
            continue
        G = groups[key]
        members = [glob(r) for r in key]
        _replicate_children(dist, G, grank, members, nd, rs, glob, backend, n, inf, stats)
        U, L = nd.upper.table, nd.lower.table
        w1 = min(nd.rows, n) + 1
        out = {"reach": backend.empty((n1, w1)), "trace": backend.empty((n1, w1)),
               "kmax": backend.empty((n1,)), "wstar_dev": backend.empty((1,))}
        out["wstar_dev"].zero_()
        spans = split_rows(U["kmax_host"] + 1, len(key))  # identical on every member
        lo, hi = spans[key.index(rank)]
        backend.combine_rows(U, L, out, lo, hi, inf)
        out["wstar_part"] = out["wstar_dev"]
        out["my_span"] = (lo, hi)
        out["spans"] = [(members[t], a, b) for t, (a, b) in enumerate(spans)]
        nd.table = out
    ctx = {"rs": rs, "groups": groups, "glob": glob, "group": group, "stats": stats}
    return root, bands, upper, ctx


def recover_sharded(root: Node, bands: List[Node], m: int, dist, group=None, backend=None,
                    ctx=None):
    """Cross-vertex columns of the LCS path (solver.py:180-207), stitched from
    the upper-level walk and the band walks.  Each rank walks only the path
    towards its own band: at a node, the owner of the trace row broadcasts
    (k, x) within the node's group; then every member follows the child
    whose subtree holds it.  The band pieces and the path's end column are
    merged with one max all-reduce of an (m+1) int32 vector (columns >= 1)."""
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
            k = nd.table["trace"][i - 1, jj]
            kx[0] = k
            kx[1] = nd.upper.table["reach"][i - 1, k]
        _bcast(dist, G, kx, owner)
        k, x = (int(v) for v in kx.cpu().tolist())
        if rank in rs[id(nd.upper)]:
            walk(nd.upper, i, k)
        if rank in rs[id(nd.lower)]:
            walk(nd.lower, x, jj - k)

    if rank in rs[id(root)]:
        walk(root, 1, length)
    path = backend.empty((m + 1,))
    path.zero_()
    for b in bands:
        if b.band % P == rank:
            i, jj = start[b.band]
            seg = backend.recover_band(b.table["handle"], i, jj, b.rows)
            path[b.top - 1: b.top - 1 + len(seg)].copy_(torch.from_numpy(seg))
    # the path's end column: root cell (start column 1, weight length), held by
    # the owner of row 0 (root rows are not replicated)
    if R is not None and grank == r0:
        path[m: m + 1].copy_(R["reach"][0, length].reshape(1))
    _all_reduce_max(dist, group, path)
    return length, path.cpu().numpy().astype(np.int32)


def lcs_sharded(a, b, *, group=None, device=None, low_memory=False, backend=None,
                stats: Optional[CommStats] = None) -> LcsResult:
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
                                                with_trace=not low_memory, stats=stats)
        length, path = recover_sharded(root, bands, len(rows), dist, group, backend, ctx)
    finally:
        if own:
            backend.free()
    r = backend.assemble(GridModel(rows, cols), path)
    if swapped:
        r = LcsResult(r.length, r.subsequence, r.col_positions, r.row_positions)
    return r
