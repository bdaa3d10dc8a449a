"""Pin the C oracle (the parity checker) before trusting it (CPU only).

Checks oracle/lcsgrid_oracle.c against every golden the reference offers for
this path: SPEC known answers, the paper grid (every node), whole trees and
lcs() outputs of the real reference (tests/golden/, made by make_golden.py),
the full-size config digests, and -- when oracle/_ref was built here -- the
reference itself on fresh random instances.
"""

import hashlib

import numpy as np
import pytest

import oracle as O
import workloads

PAPER_COLS, PAPER_ROWS = "gatttatgcagg", "tcaggatt"


def test_spec_base_case_rows(spec_examples):
    for key in ("base_case_row_paper", "base_case_row_ttt", "base_case_row_absent"):
        ex = spec_examples[key]
        sym = ex["rows"].encode()[ex["h"] - 1]
        assert O.base_case_row(ex["cols"], sym).tolist() == ex["expect"], key


def test_spec_paper_grid(spec_examples):
    t = O.OracleTree(PAPER_ROWS, PAPER_COLS)
    root = t.node(t.root)
    assert root.reach[0].tolist() == spec_examples["paper_row1"]["expect"]
    assert int(root.kmax[0]) == spec_examples["paper_length"]
    path = t.recover(5)
    assert int(path[-1]) == spec_examples["paper_end_column"]
    assert t.recover(0).tolist() == [1] * 9
    assert int(root.reach[0, 3]) == spec_examples["paper_reach_j3"]
    for key in ("empty", "identical", "disjoint"):
        ex = spec_examples[key]
        assert O.lcs(ex["a"], ex["b"])[0] == ex["length"]


def _compare_tree(tree, nodes, with_trace=True):
    assert len(tree) == len(nodes)
    for idx, exp in enumerate(nodes):
        got = tree.node(idx)
        assert (got.top_row, got.bottom_row) == (exp["top"], exp["bottom"]), idx
        np.testing.assert_array_equal(got.reach, exp["reach"])
        np.testing.assert_array_equal(got.kmax, exp["kmax"])
        assert got.wstar == exp["wstar"]
        if with_trace and exp["trace"] is not None:
            np.testing.assert_array_equal(got.trace, exp["trace"])


def test_paper_grid_every_node(paper_tree):
    trees, _, extra = paper_tree
    _compare_tree(O.OracleTree(PAPER_ROWS, PAPER_COLS), trees["paper"])
    import json
    exp = json.loads(bytes(extra["paper/lcs"]).decode())
    n, sub, pa, pb = O.lcs(PAPER_COLS, PAPER_ROWS)
    assert (n, sub.hex(), list(pa), list(pb)) == (
        exp["length"], exp["subsequence"], exp["row_positions"], exp["col_positions"])


def test_reference_trees(ref_trees):
    trees, meta, _ = ref_trees
    for idx, mt in enumerate(meta):
        t = O.OracleTree(bytes.fromhex(mt["rows"]), bytes.fromhex(mt["cols"]), mt["top"],
                         mt["bottom"])
        _compare_tree(t, trees[f"t{idx}"])


def test_reference_cfg1_tree(ref_trees):
    trees, _, _ = ref_trees
    a, b = workloads.generate(1)
    _compare_tree(O.OracleTree(a, b, threads=4), trees["cfg1"])


def test_reference_lcs_pairs(ref_lcs_pairs):
    for p in ref_lcs_pairs:
        a, b = bytes.fromhex(p["a"]), bytes.fromhex(p["b"])
        for low in (False, True):
            n, sub, pa, pb = O.lcs(a, b, low_memory=low)
            assert (n, sub.hex(), list(pa), list(pb)) == (
                p["length"], p["subsequence"], p["row_positions"], p["col_positions"])


@pytest.mark.parametrize("key", ["cfg1/seed0", "cfg1/seed1", "cfg2/seed0"])
def test_config_digests(config_digests, key):
    cfg, seed = int(key[3]), int(key.split("seed")[1])
    exp = config_digests[key]
    a, b = workloads.generate(cfg, seed)
    n, sub, pa, pb = O.lcs(a, b, threads=4)
    assert n == exp["length"]
    assert hashlib.sha256(sub).hexdigest() == exp["subsequence_sha256"]
    pos = np.array(pa + pb, dtype=np.int64).tobytes()
    assert hashlib.sha256(pos).hexdigest() == exp["positions_sha256"]
    rows, cols = (b, a) if len(a) > len(b) else (a, b)
    t = O.OracleTree(rows, cols, with_trace=False, threads=4, count=True)
    assert hashlib.sha256(t.node(t.root).reach.tobytes()).hexdigest() == exp["dg_sha256"]
    assert t.counters() == exp["counters"]


def test_generators_expected_lengths():
    a, b = workloads.generate(1)
    assert O.lcs(a, b)[0] == workloads.EXPECTED_LCS_SEED0[1]
    for cfg, (m, n) in {2: (2048, 2048), 3: (4096, 4096), 4: (1024, 65536),
                        5: (16384, 16384)}.items():
        a, b = workloads.generate(cfg)
        assert (len(a), len(b)) == (m, n) or (cfg == 2 and len(a) == m)


def test_against_reference_fresh(reference):
    """The oracle restatement equals the real reference (Cython backend) on
    fresh instances, every node of every tree (incl. INF-cell traces)."""
    from lcsgrid_ref import seqcore as Rs, solver as Rv

    rng = np.random.default_rng(7)
    for _ in range(40):
        m, n = int(rng.integers(1, 60)), int(rng.integers(0, 90))
        a, b = workloads.random_pair(rng, m, n, int(rng.choice([2, 4, 26])))
        g = Rs.GridModel(a, b)
        tab = Rv.build_cost_table(g, 1, m + 1)
        t = O.OracleTree(a, b)
        root = t.node(t.root)
        np.testing.assert_array_equal(root.reach, tab.reach)
        np.testing.assert_array_equal(root.trace, tab.trace)
        r = reference.lcs(a, b)
        assert O.lcs(a, b) == (r.length, r.subsequence, r.row_positions, r.col_positions)
