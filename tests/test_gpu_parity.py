"""Parity of the CUDA path (through the C-ABI) against the oracle / reference
goldens -- the parity tests proper.  Bit-exact: integer work.

Every comparison below is against (a) fixtures produced by the REAL
reference (tests/golden/, make_golden.py) or (b) the C oracle, which
tests/test_oracle.py pins to those fixtures.
"""

import ctypes
import hashlib
import json

import numpy as np
import pytest

import oracle as O
import paper_2309_09072_b200 as L
import workloads
from paper_2309_09072_b200 import _lib

pytestmark = pytest.mark.gpu

PAPER_COLS, PAPER_ROWS = "gatttatgcagg", "tcaggatt"


def gpu_tree_nodes(table):
    """Post-order (upper, lower, self) list of a device CostTable tree."""
    out = []

    def rec(t):
        if t.upper is not None:
            rec(t.upper)
            rec(t.lower)
        out.append(t)

    rec(table)
    return out


def compare_nodes(gpu_nodes, exp_nodes, trace=True):
    assert len(gpu_nodes) == len(exp_nodes)
    for idx, (g, e) in enumerate(zip(gpu_nodes, exp_nodes)):
        assert (g.top_row, g.bottom_row) == (e["top"], e["bottom"]), idx
        np.testing.assert_array_equal(g.reach, e["reach"], err_msg=f"reach node {idx}")
        np.testing.assert_array_equal(g.kmax, e["kmax"], err_msg=f"kmax node {idx}")
        assert g.wstar == e["wstar"], idx
        if trace and e["trace"] is not None:
            np.testing.assert_array_equal(g.trace, e["trace"], err_msg=f"trace node {idx}")


def test_device_visible():
    assert _lib.load().lcsg_device_count() >= 1


def test_paper_grid(paper_tree, spec_examples):
    trees, _, extra = paper_tree
    g = L.GridModel(PAPER_ROWS, PAPER_COLS)
    tab = L.build_cost_table(g, 1, g.m + 1)
    compare_nodes(gpu_tree_nodes(tab), trees["paper"])
    assert L.lcs_length(tab) == spec_examples["paper_length"]
    assert int(L.recover_cross_vertices(g, tab, 5)[-1]) == spec_examples["paper_end_column"]
    assert L.recover_cross_vertices(g, tab, 0).tolist() == [1] * 9
    exp = json.loads(bytes(extra["paper/lcs"]).decode())
    r = L.lcs(PAPER_COLS, PAPER_ROWS)
    assert (r.length, r.subsequence.hex(), list(r.row_positions), list(r.col_positions)) == (
        exp["length"], exp["subsequence"], exp["row_positions"], exp["col_positions"])


def test_reference_trees_every_node(ref_trees):
    trees, meta, _ = ref_trees
    for idx, mt in enumerate(meta):
        g = L.GridModel(bytes.fromhex(mt["rows"]), bytes.fromhex(mt["cols"]))
        tab = L.build_cost_table(g, mt["top"], mt["bottom"])
        compare_nodes(gpu_tree_nodes(tab), trees[f"t{idx}"])


def test_reference_cfg1_tree_every_node(ref_trees):
    trees, _, _ = ref_trees
    a, b = workloads.generate(1)
    g = L.GridModel(a, b)
    compare_nodes(gpu_tree_nodes(L.build_cost_table(g, 1, g.m + 1)), trees["cfg1"])


@pytest.mark.parametrize("key64", ["0", "1"])
def test_reference_lcs_pairs(ref_lcs_pairs, key64, monkeypatch):
    monkeypatch.setenv("LCSG_FORCE_KEY64", key64)
    for p in ref_lcs_pairs:
        a, b = bytes.fromhex(p["a"]), bytes.fromhex(p["b"])
        for low in (False, True):
            r = L.lcs(a, b, low_memory=low)
            assert (r.length, r.subsequence.hex(), list(r.row_positions),
                    list(r.col_positions)) == (p["length"], p["subsequence"],
                                               p["row_positions"], p["col_positions"]), (p, low)


def test_random_against_oracle_trees():
    rng = np.random.default_rng(11)
    for it in range(60):
        m = int(rng.integers(1, 200))
        n = int(rng.integers(0, 300))
        sigma = int(rng.choice([2, 4, 20, 26, 200]))
        a, b = workloads.random_pair(rng, m, n, sigma, base=int(rng.integers(0, 50)))
        g = L.GridModel(a, b)
        tab = L.build_cost_table(g, 1, m + 1)
        t = O.OracleTree(a, b)
        root = t.node(t.root)
        np.testing.assert_array_equal(tab.reach, root.reach)
        if root.trace is not None:
            np.testing.assert_array_equal(tab.trace, root.trace)
        np.testing.assert_array_equal(tab.kmax, root.kmax)
        length = L.lcs_length(tab)
        assert length == int(root.kmax[0])
        for j in sorted({0, length, length // 2, max(0, length - 1)}):
            np.testing.assert_array_equal(L.recover_cross_vertices(g, tab, j), t.recover(j))


def test_layout_reuse_across_solves(monkeypatch):
    """The host reuses the tree + table layout of the previous solve when the
    shape and the layout knobs repeat: interleave repeated shapes with new
    data, the other trace mode, other slabs and another skeleton stride."""
    rng = np.random.default_rng(13)
    pairs = [workloads.random_pair(rng, 150, 190, s) for s in (4, 26, 4)]
    t_full = [O.OracleTree(a, b) for a, b in pairs]
    for stride in (None, "1", None):
        if stride is None:
            monkeypatch.delenv("LCSG_SKELETON_STRIDE", raising=False)
        else:
            monkeypatch.setenv("LCSG_SKELETON_STRIDE", stride)
        for (a, b), t in zip(pairs, t_full):
            g = L.GridModel(a, b)
            for with_trace in (True, True, False):
                tab = L.build_cost_table(g, 1, 151, with_trace=with_trace)
                np.testing.assert_array_equal(tab.reach, t.node(t.root).reach)
                length = L.lcs_length(tab)
                np.testing.assert_array_equal(L.recover_cross_vertices(g, tab, length),
                                              t.recover(length))
            sub = L.build_cost_table(g, 40, 101)  # another slab, then the full grid again
            ref = O.OracleTree(a, b, 40, 101)
            np.testing.assert_array_equal(sub.reach, ref.node(ref.root).reach)
            np.testing.assert_array_equal(sub.trace, ref.node(ref.root).trace)


def test_low_memory_tables_and_retrace():
    rng = np.random.default_rng(12)
    for _ in range(20):
        m, n = int(rng.integers(2, 150)), int(rng.integers(2, 200))
        a, b = workloads.random_pair(rng, m, n, int(rng.choice([2, 4, 26])))
        g = L.GridModel(a, b)
        lo = L.build_cost_table(g, 1, m + 1, with_trace=False)
        hi = L.build_cost_table(g, 1, m + 1, with_trace=True)
        assert lo.trace is None
        np.testing.assert_array_equal(lo.reach, hi.reach)
        length = L.lcs_length(lo)
        for j in (0, length):
            np.testing.assert_array_equal(L.recover_cross_vertices(g, lo, j),
                                          L.recover_cross_vertices(g, hi, j))


def test_edge_cases():
    # n = 0 -> D_G [[1]]; m = 1 single leaf; m > n direct build
    g = L.GridModel("abc", "")
    tab = L.build_cost_table(g, 1, 4)
    assert tab.reach.tolist() == [[1]]
    g = L.GridModel("a", "xax")
    tab = L.build_cost_table(g, 1, 2)
    assert tab.reach.tolist() == [[1, 3], [2, 3], [3, 5], [4, 5]]
    assert L.recover_cross_vertices(g, tab, 1).tolist() == [1, 3]
    for a, b in (("zzzzzzzz", "zz"), ("abcdefgh", "hgf"), ("a" * 70, "a" * 90)):
        g = L.GridModel(a, b)
        t = O.OracleTree(a, b)
        np.testing.assert_array_equal(L.build_cost_table(g, 1, g.m + 1).reach,
                                      t.node(t.root).reach)
    assert L.lcs("abcabba", "abcabba").subsequence == b"abcabba"
    assert L.lcs("abcd", "efgh").length == 0
    full = bytes(range(256))
    r = L.lcs(full, full[::-1] + full)
    assert r.length == 256 and r.subsequence == full
    g = L.GridModel(PAPER_ROWS, PAPER_COLS)
    tab = L.build_cost_table(g, 1, g.m + 1)
    with pytest.raises(ValueError, match="no path of weight 6"):
        L.recover_cross_vertices(g, tab, 6)
    sub = L.build_cost_table(g, 2, 6)
    with pytest.raises(ValueError, match="full-grid"):
        L.recover_cross_vertices(g, sub, 1)


def test_kernel_mirrors():
    import torch

    rng = np.random.default_rng(5)
    for _ in range(10):
        n = int(rng.integers(1, 500))
        cols = workloads.random_pair(rng, 1, n, 4)[1]
        d_cols = torch.from_numpy(np.frombuffer(cols, dtype=np.uint8).copy()).cuda()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        for sym in b"abcz":
            rc = _lib.load().lcsg_base_case_row(d_cols.data_ptr(), n, sym, out.data_ptr(), None)
            _lib.check(rc)
            np.testing.assert_array_equal(out.cpu().numpy(), O.base_case_row(cols, sym))
    # combine_level mirror on real upper/lower tables of an oracle tree
    for _ in range(6):
        m, n = int(rng.integers(4, 120)), int(rng.integers(4, 260))
        a, b = workloads.random_pair(rng, m, n, int(rng.choice([2, 4, 26])))
        t = O.OracleTree(a, b)
        root = t.node(t.root)
        U, Lo = t.node(root.upper), t.node(root.lower)
        exp_r, exp_t, _ = O.combine_level(U.reach, U.kmax, Lo.reach, Lo.wstar, root.reach.shape[1],
                                          t.inf)
        dU = torch.from_numpy(U.reach).cuda()
        dK = torch.from_numpy(U.kmax).cuda()
        dL = torch.from_numpy(Lo.reach).cuda()
        r = torch.zeros_like(torch.from_numpy(exp_r)).cuda()
        tr = torch.zeros_like(r)
        i_lo, i_hi = 1, n + 1
        rc = _lib.load().lcsg_combine_level(
            dU.data_ptr(), U.reach.shape[1], dK.data_ptr(), dL.data_ptr(), Lo.reach.shape[1],
            Lo.wstar, r.data_ptr(), tr.data_ptr(), exp_r.shape[1], 1, t.inf, n + 1, i_lo, i_hi,
            None)
        _lib.check(rc)
        np.testing.assert_array_equal(r.cpu().numpy()[i_lo:i_hi], exp_r[i_lo:i_hi])
        np.testing.assert_array_equal(tr.cpu().numpy()[i_lo:i_hi], exp_t[i_lo:i_hi])


def test_assemble_and_device_view():
    rng = np.random.default_rng(6)
    for _ in range(10):
        m, n = int(rng.integers(1, 90)), int(rng.integers(1, 120))
        a, b = workloads.random_pair(rng, m, n, 4)
        g = L.GridModel(a, b)
        tab = L.build_cost_table(g, 1, m + 1)
        path = L.recover_cross_vertices(g, tab, L.lcs_length(tab))
        r = L.assemble_lcs(g, path)
        assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.assemble(a, b, path)
        np.testing.assert_array_equal(tab.reach_device.cpu().numpy(), tab.reach)


def gpu_tree_digest(table) -> str:
    """tree_digest() of tests/golden/make_deep_digests.py over a device tree:
    node ids are the reference's post-order creation ids, so records are
    hashed in id order; buffers are reused (one node on the host at a time)."""
    from make_deep_digests import node_record

    lib = _lib.load()
    h = table._tree.handle
    acc = hashlib.sha256()
    info = (ctypes.c_int32 * 8)()
    buf = np.empty(0, np.int32)
    for node in range(lib.lcsg_num_nodes(h)):
        _lib.check(lib.lcsg_node_info(h, node, info))
        w1, upper, n = info[2], info[3], info[6]
        cells = (n + 1) * w1
        if buf.size < 2 * cells + n + 1:
            buf = np.empty(2 * cells + n + 1, np.int32)
        reach = buf[:cells]
        kmax = buf[2 * cells:2 * cells + n + 1]
        _lib.check(lib.lcsg_node_reach(h, node, reach.ctypes.data))
        _lib.check(lib.lcsg_node_kmax(h, node, kmax.ctypes.data))
        trace = None
        if upper >= 0:
            trace = buf[cells:2 * cells]
            _lib.check(lib.lcsg_node_trace(h, node, trace.ctypes.data))
        w = ctypes.c_int32()
        _lib.check(lib.lcsg_node_wstar(h, node, ctypes.byref(w)))
        acc.update(node_record(reach, trace, kmax, w.value))
    return acc.hexdigest()


def _check_lcs_digest(exp, a, b, low_memory):
    r = L.lcs(a, b, low_memory=low_memory)
    assert r.length == exp["length"], low_memory
    assert hashlib.sha256(r.subsequence).hexdigest() == exp["subsequence_sha256"], low_memory
    pos = np.array(r.row_positions + r.col_positions, dtype=np.int64).tobytes()
    assert hashlib.sha256(pos).hexdigest() == exp["positions_sha256"], low_memory


def _check_digest(exp, a, b, low_memory_too=False, deep=True):
    """lcs() in TRACED mode (the path bench.py times) and, optionally,
    low-memory mode; the final D_G built with and without traces; the final
    trace table and every node of the traced tree when the reference digests
    hold them (tests/golden/make_deep_digests.py)."""
    _check_lcs_digest(exp, a, b, low_memory=False)
    if low_memory_too:
        _check_lcs_digest(exp, a, b, low_memory=True)
    rows, cols = (b, a) if len(a) > len(b) else (a, b)
    g = L.GridModel(rows, cols)
    tab = L.build_cost_table(g, 1, g.m + 1, with_trace=False)
    assert hashlib.sha256(tab.reach.tobytes()).hexdigest() == exp["dg_sha256"]
    del tab
    tab = L.build_cost_table(g, 1, g.m + 1, with_trace=True)
    assert hashlib.sha256(tab.reach.tobytes()).hexdigest() == exp["dg_sha256"]
    if "trace_sha256" in exp:
        assert hashlib.sha256(tab.trace.tobytes()).hexdigest() == exp["trace_sha256"]
    if deep and "tree_sha256" in exp:
        assert gpu_tree_digest(tab) == exp["tree_sha256"]


DIGEST_KEYS = [f"cfg{c}/seed{s}" for c in (1, 2, 3, 4, 5) for s in (0, 1, 2)]


@pytest.mark.parametrize("key", DIGEST_KEYS)
def test_config_digests(config_digests, key):
    """Every config, seeds 0-2, against the reference's own digests: traced
    lcs() (what bench.py times), low-memory lcs() on cfg4/cfg5, D_G in both
    trace modes, the final trace table and a digest of every node of the
    traced tree (reach, trace, kmax, wstar)."""
    if key not in config_digests:
        pytest.skip(f"{key} digest not generated")
    cfg, seed = int(key[3]), int(key.split("seed")[1])
    a, b = workloads.generate(cfg, seed)
    _check_digest(config_digests[key], a, b, low_memory_too=(cfg >= 4))


@pytest.mark.parametrize("key", ["cfg1/seed0", "cfg2/seed1", "cfg3/seed2", "cfg4/seed0"])
def test_config_digests_key64(config_digests, key, monkeypatch):
    """The 64-bit packed-key instantiation of every kernel (selected at
    bits(n+2) + bits(max k) > 32, e.g. 100k x 100k inputs) forced on at
    config scale: same digests, every node of the tree included."""
    monkeypatch.setenv("LCSG_FORCE_KEY64", "1")
    cfg, seed = int(key[3]), int(key.split("seed")[1])
    a, b = workloads.generate(cfg, seed)
    _check_digest(config_digests[key], a, b, low_memory_too=True)


def _dg_row_by_definition(rows: bytes, cols: bytes, i: int, w1: int) -> np.ndarray:
    """Independent D_G row: D(i,j) = i + min{t :
    LCS(rows, cols[i-1:i-1+t]) >= j}, INF if none -- one numpy DP sweep."""
    from paper_2309_09072_b200.dp import _table
    n = len(cols)
    H = _table(rows, cols[i - 1:])[-1]  # H[t] = LCS(rows, cols[i-1:i-1+t])
    out = np.full(w1, n + 2, dtype=np.int64)
    for j in range(w1):
        hit = np.flatnonzero(H >= j)
        if len(hit):
            out[j] = i + hit[0]
    return out


@pytest.mark.parametrize("cfg", [2, 3])
def test_dg_rows_by_definition(cfg):
    """Size-independent property at config scale: random rows of the final
    D_G equal the breakout definition computed by a plain DP."""
    a, b = workloads.generate(cfg)
    rows, cols = (b, a) if len(a) > len(b) else (a, b)
    g = L.GridModel(rows, cols)
    tab = L.build_cost_table(g, 1, g.m + 1, with_trace=False)
    R = tab.reach
    rng = np.random.default_rng(cfg)
    for i in [1, len(cols) + 1] + [int(x) for x in rng.integers(1, len(cols) + 2, 3)]:
        np.testing.assert_array_equal(R[i - 1], _dg_row_by_definition(rows, cols, i, R.shape[1]))


@pytest.mark.parametrize("sweep", ["0", "1"])
@pytest.mark.parametrize("stride", [1, 2, 4, 16, 64, 512])
def test_skeleton_refine_strides(stride, sweep, monkeypatch):
    """The wide-table combine (skeleton rows by exact bisection + the row sweep,
    or with LCSG_SWEEP=0 the refinement passes bounded by neighbouring rows) is
    bit-exact -- reach, kmax, wstar and every trace cell incl. INF artifacts --
    for any skeleton stride."""
    monkeypatch.setenv("LCSG_SWEEP", sweep)
    monkeypatch.setenv("LCSG_SKELETON_STRIDE", str(stride))
    monkeypatch.setenv("LCSG_SWEEP_STRIDE", str(max(2, stride)))
    rng = np.random.default_rng(100 + stride)
    for _ in range(12):
        m = int(rng.integers(66, 330))
        n = int(rng.integers(40, 420))
        sigma = int(rng.choice([2, 4, 20, 26]))
        a, b = workloads.random_pair(rng, m, n, sigma)
        g = L.GridModel(a, b)
        t = O.OracleTree(a, b)
        for with_trace in (True, False):
            tab = L.build_cost_table(g, 1, m + 1, with_trace=with_trace)
            nodes = gpu_tree_nodes(tab)
            for idx in range(len(t)):
                exp = t.node(idx)
                if exp.upper < 0:
                    continue
                got = nodes[idx]
                np.testing.assert_array_equal(got.reach, exp.reach, err_msg=f"S={stride} {idx}")
                np.testing.assert_array_equal(got.kmax, exp.kmax)
                assert got.wstar == exp.wstar
                if with_trace:
                    np.testing.assert_array_equal(got.trace, exp.trace, err_msg=f"S={stride} {idx}")
            length = L.lcs_length(tab)
            np.testing.assert_array_equal(L.recover_cross_vertices(g, tab, length),
                                          t.recover(length))


@pytest.mark.parametrize("key64", ["0", "1"])
@pytest.mark.parametrize("env", [
    {"LCSG_SKELETON_STRIDE": "64", "LCSG_COL_BLOCK": "8", "LCSG_SWEEP": "0"},   # two stages: step 8, step 1
    {"LCSG_SKELETON_STRIDE": "32", "LCSG_COL_BLOCK": "4", "LCSG_SWEEP": "0"},   # stages: step 8, 2, 1 (B=4,4,2)
    {"LCSG_SKELETON_STRIDE": "8", "LCSG_COL_BLOCK": "2", "LCSG_SWEEP": "0"},    # three stages of B=2
    {"LCSG_SKELETON_STRIDE": "32", "LCSG_COL_BLOCK": "32", "LCSG_SWEEP": "0"},  # one stage of 32 rows
    {"LCSG_REFINE_PASSES": "1", "LCSG_SWEEP": "0"},                            # one launch per refinement pass
    {"LCSG_THREAD_MAX_W1": "3", "LCSG_SKEL_THREAD_MAX_W1": "3", "LCSG_SKEL_WARP_MAX_W1": "9"},
    {"LCSG_SKEL_THREAD_MAX_W1": "1", "LCSG_SKEL_WARP_MAX_W1": "1"},  # CTA kernel for every skeleton row
    {"LCSG_NARROW": "0"},                                   # bisection kernel for the narrow tables
    {"LCSG_THREAD_MAX_W1": "33"},                           # 65-wide tables through the column path
    {"LCSG_LEAFPAIR": "0"},                                 # height-1 combines through the staged kernel
    {"LCSG_NARROW": "0", "LCSG_THREAD_MAX_W1": "65"},
    {"LCSG_NARROW32_ROLL": "0"},                            # unrolled-fold narrow<32> kernel
    {"LCSG_FINE_SC_MAXW1": "0", "LCSG_SWEEP": "0"},                            # runtime block size in the fine kernel
    {"LCSG_SKELETON_STRIDE": "512", "LCSG_COL_BLOCK": "8", "LCSG_SWEEP": "0"},  # row-step 64 / 8 / 1 stages
    {"LCSG_SKEL_WARP_BATCHED": "0"},                        # per-node warp DFS for w1 <= 257 skeletons
    {"LCSG_NARROW_FW": "0"},                                # narrow kernels with a runtime row width
    {"LCSG_VIRTUAL_H1": "0"},                               # height-1 tables materialised (leaf-pair kernel)
    {"LCSG_VIRTUAL_H1": "0", "LCSG_LEAFPAIR": "0"},         # ... and computed by the staged narrow kernel
])
def test_refinement_variants(env, key64, monkeypatch):
    """Every geometry / schedule of the wide-table combine is bit-exact, with
    32-bit and (forced) 64-bit packed keys."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("LCSG_FORCE_KEY64", key64)
    import zlib

    rng = np.random.default_rng(zlib.crc32(repr(sorted(env.items())).encode()))
    for _ in range(8):
        m = int(rng.integers(40, 300))
        n = int(rng.integers(20, 500))
        sigma = int(rng.choice([2, 4, 26]))
        a, b = workloads.random_pair(rng, m, n, sigma)
        g = L.GridModel(a, b)
        t = O.OracleTree(a, b)
        nodes = gpu_tree_nodes(L.build_cost_table(g, 1, m + 1))
        for idx in range(len(t)):
            exp = t.node(idx)
            if exp.upper < 0:
                continue
            np.testing.assert_array_equal(nodes[idx].reach, exp.reach, err_msg=f"{env} {idx}")
            np.testing.assert_array_equal(nodes[idx].trace, exp.trace, err_msg=f"{env} {idx}")
            np.testing.assert_array_equal(nodes[idx].kmax, exp.kmax)
            assert nodes[idx].wstar == exp.wstar


def test_skeleton_cta_wide_rows(monkeypatch):
    """The CTA-per-row skeleton kernel on long rows (batched per-warp DFS with
    many nodes per batch, so the largest finite column is found by lanes other
    than lane 0): every node's kmax, wstar, reach and trace stay bit-exact."""
    monkeypatch.setenv("LCSG_SKEL_THREAD_MAX_W1", "1")
    monkeypatch.setenv("LCSG_SKEL_WARP_MAX_W1", "1")
    rng = np.random.default_rng(777)
    for m, n, sigma in ((300, 2500, 26), (520, 1800, 4), (260, 3100, 20)):
        a, b = workloads.random_pair(rng, m, n, sigma)
        g = L.GridModel(a, b)
        t = O.OracleTree(a, b)
        nodes = gpu_tree_nodes(L.build_cost_table(g, 1, m + 1))
        for idx in range(len(t)):
            exp = t.node(idx)
            if exp.upper < 0:
                continue
            np.testing.assert_array_equal(nodes[idx].kmax, exp.kmax, err_msg=f"{m}x{n} {idx}")
            assert nodes[idx].wstar == exp.wstar
            np.testing.assert_array_equal(nodes[idx].reach, exp.reach, err_msg=f"{m}x{n} {idx}")
            np.testing.assert_array_equal(nodes[idx].trace, exp.trace, err_msg=f"{m}x{n} {idx}")


def test_narrow_window_overflow():
    """Sparse matches (256 symbols, long columns): the reach of a 16-row slab
    runs far past the narrow kernel's staged L window, so its direct-read path
    is exercised; every node stays bit-exact."""
    rng = np.random.default_rng(4242)
    for m, n in ((64, 6000), (40, 9000), (33, 3000)):
        a = rng.integers(0, 256, m).astype(np.uint8).tobytes()
        b = rng.integers(0, 256, n).astype(np.uint8).tobytes()
        g = L.GridModel(a, b)
        t = O.OracleTree(a, b)
        nodes = gpu_tree_nodes(L.build_cost_table(g, 1, m + 1))
        for idx in range(len(t)):
            exp = t.node(idx)
            if exp.upper < 0:
                continue
            np.testing.assert_array_equal(nodes[idx].reach, exp.reach, err_msg=f"{m}x{n} {idx}")
            np.testing.assert_array_equal(nodes[idx].trace, exp.trace, err_msg=f"{m}x{n} {idx}")
            np.testing.assert_array_equal(nodes[idx].kmax, exp.kmax)
            assert nodes[idx].wstar == exp.wstar
        r = L.lcs(a, b)
        assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b)


def test_lcs_many_matches_sequential():
    """Overlapped independent solves (lcs_many) return exactly the sequential
    results, in order, for mixed sizes, alphabets and empty inputs."""
    rng = np.random.default_rng(99)
    pairs = [workloads.random_pair(rng, int(rng.integers(1, 300)), int(rng.integers(1, 400)),
                                   int(rng.choice([2, 4, 26]))) for _ in range(40)]
    pairs += [(b"", b"abc"), (b"gatttatgcagg", b"tcaggatt"), workloads.generate(1)]
    got = L.lcs_many(pairs, concurrency=8)
    assert got == [L.lcs(a, b) for a, b in pairs]
    for (a, b), r in zip(pairs[:10], got[:10]):
        assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b)
    assert L.lcs_many(pairs[:5], concurrency=1, low_memory=True) == got[:5]


@pytest.mark.parametrize("low", [False, True])
def test_lcs_batch_equal_shapes(low):
    """Batched solve (one launch per tree height for all pairs, SURVEY.md
    8(f) rank 4) == the per-pair solves == the oracle, for equal-shape groups
    incl. swapped orientation, m = 1 (leaf roots), n = 1, sparse alphabets and
    identical / disjoint pairs."""
    rng = np.random.default_rng(4040)
    shapes = [(37, 120, 4), (120, 37, 26), (1, 50, 2), (50, 1, 2), (64, 64, 4), (300, 420, 20),
              (2, 2, 2), (3, 9, 3)]
    for la, lb, sigma in shapes:
        pairs = [workloads.random_pair(rng, la, lb, sigma) for _ in range(5)]
        if la == lb:
            pairs.append((pairs[0][0], pairs[0][0]))
        got = L.lcs_batch([a for a, _ in pairs], [b for _, b in pairs], low_memory=low)
        for (a, b), r in zip(pairs, got):
            assert r == L.lcs(a, b, low_memory=low), (la, lb)
            assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b)


def test_lcs_batch_cfg4_windows(config_digests):
    """cfg4's query against a window around each of its 8 planted copies, as
    one batched solve: bit-exact against the sequential solves and the oracle."""
    pairs = workloads.cfg4_planted_windows(0, width=4096)
    got = L.lcs_batch([a for a, _ in pairs], [b for _, b in pairs])
    for (a, b), r in zip(pairs, got):
        assert r == L.lcs(a, b)
        assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b, threads=8)
    assert L.lcs_many(pairs + [(b"ab", b"b")]) == got + [L.lcs(b"ab", b"b")]


def test_lcs_batch_errors():
    with pytest.raises(ValueError, match="equal shape"):
        L.lcs_batch([b"ab", b"abc"], [b"x", b"y"])
    assert L.lcs_batch([], []) == []
    assert L.lcs_batch([b"", b""], [b"a", b"b"]) == [L.LcsResult(0, b"", (), ())] * 2


def test_graph_replay_repeated_shapes(monkeypatch):
    """Per-shape CUDA graphs: repeated solves of one shape (new data each time)
    replay the first solve's build and walk graphs on its arena -- through
    lcs() in both modes, build_cost_table (every node via the API), batches,
    a second handle of the shape alive at the same time (normal path), knob
    changes (a new key) and lcsg_trim -- always bit-exact against the oracle."""
    rng = np.random.default_rng(2718)
    lib = _lib.load()
    for rnd in range(3):
        for low in (False, True):
            for _ in range(3):
                a, b = workloads.random_pair(rng, 90, 130, int(rng.choice([2, 4, 26])))
                r = L.lcs(a, b, low_memory=low)
                assert (r.length, r.subsequence, r.row_positions, r.col_positions) == O.lcs(a, b)
        pairs = [workloads.random_pair(rng, 40, 70, 4) for _ in range(4)]
        got = L.lcs_batch([p[0] for p in pairs], [p[1] for p in pairs])
        assert [(r.length, r.subsequence, r.row_positions, r.col_positions) for r in got] == \
            [O.lcs(a, b) for a, b in pairs]
        a, b = workloads.random_pair(rng, 70, 160, 4)
        g = L.GridModel(a, b)
        held = L.build_cost_table(g, 1, g.m + 1)  # keeps the shape's entry busy
        a2, b2 = workloads.random_pair(rng, 70, 160, 26)
        g2 = L.GridModel(a2, b2)
        second = L.build_cost_table(g2, 1, g2.m + 1)
        for tab, (x, y) in ((held, (a, b)), (second, (a2, b2))):
            t = O.OracleTree(x, y)
            nodes = gpu_tree_nodes(tab)
            for idx in range(len(t)):
                np.testing.assert_array_equal(nodes[idx].reach, t.node(idx).reach)
                if t.node(idx).trace is not None:
                    np.testing.assert_array_equal(nodes[idx].trace, t.node(idx).trace)
            length = L.lcs_length(tab)
            np.testing.assert_array_equal(L.recover_cross_vertices(L.GridModel(x, y), tab, length),
                                          t.recover(length))
        del held, second
        monkeypatch.setenv("LCSG_SKELETON_STRIDE", "16" if rnd == 0 else "8")
        if rnd == 1:
            assert lib.lcsg_trim(0) == 0


def test_reserve_and_trim():
    """Pool management entry points: reserve maps HBM into the library's pool
    up front, trim returns it (and drops idle graph-cache entries); solves
    around them stay exact."""
    a, b = workloads.generate(1)
    L.reserve(64 << 20)
    r1 = L.lcs(a, b)
    L.trim()
    assert L.lcs(a, b) == r1
    with pytest.raises(ValueError, match="negative size"):
        L.reserve(-1)
