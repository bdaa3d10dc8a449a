"""Multi-rank schedule (paper_2309_09072_b200/distributed.py).

CPU: world_size 2 and 4 over gloo with an oracle-backed backend (the C
oracle computes each band subtree and each row range of the upper combines),
so the host logic -- band plan, balanced start-column shards, row-range
broadcasts, wstar all-reduce, recovery stitching -- is checked bit-exactly
against the single-process oracle without a GPU.
GPU: 2 ranks on one B200 over gloo with the real C-ABI backend (kernels never
wait on each other; collectives are host-side), against the 1-GPU solve.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads
from paper_2309_09072_b200 import distributed as D
from paper_2309_09072_b200.seqcore import LcsResult


class OracleBackend:
    """Test-only backend: the C oracle as the 'device' (CPU torch tensors)."""

    def empty(self, shape, dtype="int32"):
        return torch.zeros(shape, dtype=torch.int32)

    def build_band(self, rows, cols, top, bottom, with_trace):
        t = O.OracleTree(rows, cols, top, bottom, with_trace=with_trace)
        r = t.node(t.root)
        return t, torch.from_numpy(r.reach.copy()), torch.from_numpy(r.kmax.copy()), r.wstar

    def combine_rows(self, U, L, out, lo, hi, inf):
        reach, trace, _ = O.combine_level(U["reach"].numpy(), U["kmax"].numpy(), L["reach"].numpy(),
                                          L["wstar"], out["reach"].shape[1], inf, True, lo, hi)
        out["reach"][lo:hi] = torch.from_numpy(reach[lo:hi])
        out["trace"][lo:hi] = torch.from_numpy(trace[lo:hi])
        if hi > lo:
            km = (reach[lo:hi] < inf).sum(1) - 1
            out["kmax"][lo:hi] = torch.from_numpy(km.astype(np.int32))
            out["wstar_dev"][0] = max(int(out["wstar_dev"][0]), int(km.max()))

    def recover_band(self, tree, i_start, j, m_band):
        nodes = tree.nodes()
        top0 = nodes[tree.root].top_row
        cols = np.zeros(m_band + 1, dtype=np.int32)

        def walk(idx, i, jj):
            nd = nodes[idx]
            if nd.upper < 0:
                cols[nd.top_row - top0] = i
                return
            U, L = nodes[nd.upper], nodes[nd.lower]
            if nd.trace is not None:
                k = int(nd.trace[i - 1, jj])
            else:  # solver.py:165-177 first-wins retrace
                best, k = tree.inf, 0
                for kk in range(min(jj, int(U.kmax[i - 1])) + 1):
                    x = int(U.reach[i - 1, kk])
                    v = tree.inf if (x >= tree.inf or jj - kk >= L.reach.shape[1]) else int(L.reach[x - 1, jj - kk])
                    if v < best:
                        best, k = v, kk
            x = int(U.reach[i - 1, k])
            walk(nd.upper, i, k)
            walk(nd.lower, x, jj - k)

        walk(tree.root, i_start, j)
        cols[m_band] = int(nodes[tree.root].reach[i_start - 1, j])
        return cols

    def synchronize(self):
        pass

    def assemble(self, g, path):
        n, sub, rp, cp = O.assemble(g.row_seq, g.col_seq, path)
        return LcsResult(n, sub, rp, cp)

    def free(self):
        pass


def _check_tables(t, root, bands, upper, rank):
    """Every table a rank holds equals the oracle's: rows it owns, and the
    full tables it received to compute a parent combine."""
    for nd in list(bands) + list(upper):
        T = nd.table
        if T is None:
            continue
        exp = t.node(_node_id(t, nd))
        reach = np.asarray(T["reach"])
        kmax = np.asarray(T["kmax"])
        if T.get("reach_full"):
            np.testing.assert_array_equal(reach, exp.reach)
            np.testing.assert_array_equal(kmax, exp.kmax)
            assert T["wstar"] == exp.wstar
        if "trace" in T:  # computed here: the rows this rank owns
            lo, hi = next((a, b) for r, a, b in T["spans"] if r == rank)
            np.testing.assert_array_equal(reach[lo:hi], exp.reach[lo:hi])
            np.testing.assert_array_equal(np.asarray(T["trace"])[lo:hi], exp.trace[lo:hi])
            np.testing.assert_array_equal(kmax[lo:hi], exp.kmax[lo:hi])
            if "wstar" in T:  # known once the node was replicated for its parent
                assert T["wstar"] == exp.wstar
    # every rank owning a band takes part in the root combine; with fewer
    # bands than ranks (short inputs) the others sit the solve out
    assert (root.table is not None) == (rank < len(bands))


def _node_id(tree, nd):
    """Oracle node id of the plan node covering vertex rows [top, bottom)."""
    for idx in range(len(tree)):
        o = tree.node(idx)
        if o.top_row == nd.top and o.bottom_row == nd.bottom:
            return idx
    raise KeyError((nd.top, nd.bottom))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cases(seed, count):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m, n = int(rng.integers(6, 110)), int(rng.integers(6, 140))
        out.append(workloads.random_pair(rng, m, n, int(rng.choice([2, 4, 26]))))
    return out


def _cpu_worker(rank, world, port, seed, count):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        be = OracleBackend()
        for a, b in _cases(seed, count):
            for low in (False, True):
                r = D.lcs_sharded(a, b, backend=be, low_memory=low)
                assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b), \
                    (a, b, low)
            rows, cols = (b, a) if len(a) > len(b) else (a, b)
            stats = D.CommStats()
            root, bands, upper, ctx = D.solve_sharded(rows, cols, dist, None, be, stats=stats)
            t = O.OracleTree(rows, cols)
            _check_tables(t, root, bands, upper, rank)
            if len(bands) > 1 and rank < len(bands):
                # every member of the root group received its sibling subtree
                assert stats.received > 0 and stats.collectives == 2 * (len(bands).bit_length() - 1)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 6), (4, 6), (8, 3)])
def test_sharded_schedule_gloo_cpu(world, count):
    mp.spawn(_cpu_worker, args=(world, _free_port(), 100 + world, count), nprocs=world, join=True)


def _subgroup_worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        G = dist.new_group([1, 2, 3])  # a proper subgroup: rank 0 sits the solves out
        if rank in (1, 2, 3):
            be = OracleBackend()
            for a, b in _cases(77, 3):
                r = D.lcs_sharded(a, b, group=G, backend=be)
                assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_schedule_proper_subgroup():
    """group= a proper subgroup of the world: only its members call into the
    schedule (their sub-subgroups use local synchronisation), and nothing hangs."""
    mp.spawn(_subgroup_worker, args=(4, _free_port()), nprocs=4, join=True)


def test_plan_and_split():
    root, bands, upper = D.build_plan(100, 8)
    assert len(bands) == 8 and len(upper) == 7 and upper[-1] is root
    assert [b.top for b in bands] == sorted(b.top for b in bands)
    assert bands[0].top == 1 and bands[-1].bottom == 101
    # too few rows: the plan shrinks to keep every band a combine (>= 2 rows)
    _, bands, _ = D.build_plan(5, 8)
    assert len(bands) == 2 and all(b.rows >= 2 for b in bands)
    spans = D.split_rows(np.array([5, 1, 1, 1, 1, 1, 1, 5]), 2)
    assert spans[0][0] == 0 and spans[-1][1] == 8 and spans[0][1] == spans[1][0]


def _gpu_worker(rank, world, port, seed, count):
    import paper_2309_09072_b200 as L

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rng = np.random.default_rng(seed)
        cases = _cases(seed, count) + [workloads.generate(1)]
        a, b = workloads.generate(2)
        cases.append((a[:900], b[:1000]))
        for a, b in cases:
            r = D.lcs_sharded(a, b, device=0)
            s = L.lcs(a, b, device=0)
            assert r == s, (len(a), len(b))
        rows, cols = workloads.generate(1)
        be = D.CudaBackend(0)
        root, bands, upper, ctx = D.solve_sharded(rows, cols, dist, None, be)
        tab = L.build_cost_table(L.GridModel(rows, cols), 1, len(rows) + 1)
        lo, hi = next((a, b) for r, a, b in root.table["spans"] if r == rank)
        np.testing.assert_array_equal(root.table["reach"].cpu().numpy()[lo:hi], tab.reach[lo:hi])
        np.testing.assert_array_equal(root.table["trace"].cpu().numpy()[lo:hi], tab.trace[lo:hi])
        be.free()
        del rng
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_schedule_two_ranks_one_gpu():
    mp.spawn(_gpu_worker, args=(2, _free_port(), 7, 6), nprocs=2, join=True)
