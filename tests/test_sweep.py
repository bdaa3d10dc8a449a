"""Parity of the row-sweep kernels (csrc/lcsg_sweep.cu) against the oracle.

The sweep generates the interior rows of every wide combine from the row
above (unit-Monge insertion structure of the tables) instead
of evaluating every cell; these tests compare EVERY node of the tree --
reach, trace incl. the INF-cell replay artefacts, kmax, wstar -- and the
recovery walk with the oracle (itself pinned to reference fixtures by
tests/test_oracle.py), for every kernel variant: register-resident warp
groups (5 / 9 / 17 cells per lane), CTA groups, the generic shared-memory /
global-state kernel, forced fallbacks, every block size, 64-bit keys.
"""

import zlib

import numpy as np
import pytest

import oracle as O
import paper_2309_09072_b200 as L
import workloads

pytestmark = pytest.mark.gpu


def gpu_tree_nodes(table):
    out = []

    def rec(t):
        if t.upper is not None:
            rec(t.upper)
            rec(t.lower)
        out.append(t)

    rec(table)
    return out


def check_pair(a, b, tag, with_trace=True):
    g = L.GridModel(a, b)
    t = O.OracleTree(a, b)
    tab = L.build_cost_table(g, 1, g.m + 1, with_trace=with_trace)
    nodes = gpu_tree_nodes(tab)
    assert len(nodes) == len(t)
    for idx in range(len(t)):
        exp = t.node(idx)
        if exp.upper < 0:
            continue
        got = nodes[idx]
        np.testing.assert_array_equal(got.reach, exp.reach, err_msg=f"{tag} reach node {idx}")
        np.testing.assert_array_equal(got.kmax, exp.kmax, err_msg=f"{tag} kmax node {idx}")
        assert got.wstar == exp.wstar, (tag, idx)
        if with_trace:
            np.testing.assert_array_equal(got.trace, exp.trace, err_msg=f"{tag} trace node {idx}")
    length = L.lcs_length(tab)
    np.testing.assert_array_equal(L.recover_cross_vertices(g, tab, length), t.recover(length))
    assert L.sweep_errors() == 0


SWEEP_ENVS = [
    {},                                                      # defaults
    {"LCSG_SWEEP_STRIDE": "2"},
    {"LCSG_SWEEP_STRIDE": "8"},
    {"LCSG_SWEEP_STRIDE": "64"},
    {"LCSG_SWEEP_STRIDE": "56"},                             # any block size, not only powers of two
    {"LCSG_SWEEP_STRIDE": "7"},
    {"LCSG_SWEEP_STRIDE": "128"},                            # longest register-kernel block
    {"LCSG_SWEEP_STRIDE": "512"},                            # beyond it: generic kernel only
    {"LCSG_SWEEP_REG": "0"},                                 # generic kernel, state in shared memory
    {"LCSG_SWEEP_REG": "0", "LCSG_SWEEP_CAP": "24"},          # ... state in the output rows (K + 2 > cap)
    {"LCSG_SWEEP_REG": "0", "LCSG_SWEEP_CPT": "1"},           # ... many threads per row
    {"LCSG_SWEEP_ONE_WARP_MAXW1": "0"},                      # CTA groups for every width
    {"LCSG_SWEEP_ONE_WARP_MAXW1": "0", "LCSG_SWEEP_GN_MAX": "64"},  # 2-warp groups; wide rows overflow -> fallback
    {"LCSG_SWEEP_CASCADE_MINLG": "7"},                       # half-size CTA groups first, flagged blocks second
    {"LCSG_SWEEP_CASCADE": "0"},
    {"LCSG_FINALIZE_SIDE": "0"},                             # finalize kernels on the handle's stream
    {"LCSG_GRAPH": "0", "LCSG_SWEEP_SMALL_CAP": "0"},         # no graph replays; uncapped CTA-group build
    {"LCSG_SWEEP_STRIDE": "16", "LCSG_THREAD_MAX_W1": "9"},   # sweep from height 4 on (events of narrow children)
    {"LCSG_SWEEP_STRIDE": "16", "LCSG_NARROW": "0", "LCSG_VIRTUAL_H1": "0"},
]


@pytest.mark.parametrize("key64", ["0", "1"])
@pytest.mark.parametrize("env", SWEEP_ENVS)
def test_sweep_variants(env, key64, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("LCSG_FORCE_KEY64", key64)
    rng = np.random.default_rng(zlib.crc32(repr(sorted(env.items())).encode()) + int(key64))
    for it in range(8):
        m = int(rng.integers(66, 700))
        n = int(rng.integers(30, 800))
        sigma = int(rng.choice([2, 4, 26]))
        a, b = workloads.random_pair(rng, m, n, sigma)
        check_pair(a, b, f"{env} {m}x{n} s{sigma}", with_trace=(it % 3 != 2))


@pytest.mark.parametrize("shape", [(1100, 2100, 26), (1300, 900, 2), (2050, 1500, 4), (300, 5000, 4)])
def test_sweep_larger_shapes(shape):
    """Multi-warp CTA groups (rows of 1025+ cells), longer walks."""
    m, n, sigma = shape
    rng = np.random.default_rng(m * 7 + n)
    a, b = workloads.random_pair(rng, m, n, sigma)
    check_pair(a, b, f"{m}x{n}")


def test_sweep_fallback_paths_are_exercised(monkeypatch):
    """The forced variants really take the paths they name: small CTA groups
    overflow on wide rows (blocks flagged, redone by the generic kernel); a tiny
    shared-memory capacity puts the row state into the output rows."""
    rng = np.random.default_rng(17)
    a, b = workloads.random_pair(rng, 900, 1200, 4)
    L.sweep_paths(reset=True)
    monkeypatch.setenv("LCSG_SWEEP_ONE_WARP_MAXW1", "0")
    monkeypatch.setenv("LCSG_SWEEP_GN_MAX", "64")
    check_pair(a, b, "overflow")
    redone, _ = L.sweep_paths(reset=True)
    assert redone > 0
    monkeypatch.delenv("LCSG_SWEEP_ONE_WARP_MAXW1")
    monkeypatch.delenv("LCSG_SWEEP_GN_MAX")
    monkeypatch.setenv("LCSG_SWEEP_REG", "0")
    monkeypatch.setenv("LCSG_SWEEP_CAP", "24")
    check_pair(a, b, "global state")
    _, glob = L.sweep_paths(reset=True)
    assert glob > 0
    monkeypatch.delenv("LCSG_SWEEP_REG")
    monkeypatch.delenv("LCSG_SWEEP_CAP")
    check_pair(a, b, "defaults")
    assert L.sweep_paths(reset=True) == (0, 0)  # the fast path handles random inputs alone


def _planted(rng, m, n, sigma, keep=0.8):
    a, b = workloads.random_pair(rng, m, n, sigma)
    k = min(m, n)
    src = np.frombuffer(a, np.uint8)[:k]
    mask = rng.random(k) < keep
    arr = np.frombuffer(b, np.uint8).copy()
    arr[:k][mask] = src[mask]
    return a, arr.tobytes()


@pytest.mark.parametrize("env", [{}, {"LCSG_SWEEP_REG": "0"}, {"LCSG_FORCE_KEY64": "1"},
                                 {"LCSG_SWEEP_REG": "0", "LCSG_SWEEP_STRIDE": "64"}])
def test_sweep_long_walks(env, monkeypatch):
    """Planted near-copies over a large alphabet: walks of hundreds of cells
    (several evaluation rounds, rounds wider than a narrow group's thread count;
    regression: the generic kernel stored / cleared only one cell per thread)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(1)
    for (m, n) in [(1530, 1414), (200, 260), (640, 700)]:
        a, b = _planted(rng, m, n, 200)
        exp = O.lcs(a, b)
        for low in (False, True):
            r = L.lcs(a, b, low_memory=low)
            assert (r.length, r.subsequence, r.row_positions, r.col_positions) == exp
    a, b = _planted(rng, 600, 640, 200)
    check_pair(a, b, f"planted {env}")


def test_sweep_cascade_second_pass(monkeypatch):
    """CTA-group cascade (half-size groups first, the blocks whose finite prefix
    overflows their registers in a second pass of full-size groups): planted
    near-copies make the upper levels' rows nearly full width."""
    monkeypatch.setenv("LCSG_SWEEP_CASCADE_MINLG", "7")
    rng = np.random.default_rng(21)
    a, b = _planted(rng, 1000, 1100, 26, keep=0.9)
    check_pair(a, b, "cascade planted")
    a, b = workloads.random_pair(rng, 1000, 1100, 2)
    check_pair(a, b, "cascade sigma 2")
    L.sweep_paths(reset=True)


def test_sweep_structured_inputs():
    """Inputs whose tables are extreme: all rows finite to full width (equal
    letters, equal strings), no match at all, periodic strings, planted copies."""
    rng = np.random.default_rng(5)
    base = (rng.integers(0, 4, 500) + 97).astype(np.uint8).tobytes()
    cases = [
        (b"a" * 300, b"a" * 420),
        (b"a" * 300, b"b" * 200),
        (base[:400], base[:400]),
        (base[:350], base[50:450]),
        (b"ab" * 200, b"ba" * 260),
        (b"abc" * 120, b"cab" * 150),
        (base[:257], base[::-1][:300]),
        (b"ab" * 100 + b"c" * 150, b"c" * 100 + b"ab" * 170),
    ]
    for i, (a, b) in enumerate(cases):
        check_pair(a, b, f"case {i}")
        check_pair(a, b, f"case {i} (no trace)", with_trace=False)


def test_sweep_matches_refinement_path(monkeypatch):
    """The sweep (default) and the column-refinement stages (LCSG_SWEEP=0) produce
    the same lcs() on a mid-size pair, and both equal the oracle."""
    rng = np.random.default_rng(99)
    a, b = workloads.random_pair(rng, 1500, 1700, 20)
    exp = O.lcs(a, b)
    for sweep in ("1", "0"):
        monkeypatch.setenv("LCSG_SWEEP", sweep)
        for low in (False, True):
            r = L.lcs(a, b, low_memory=low)
            assert (r.length, r.subsequence, r.row_positions, r.col_positions) == exp


def test_sweep_batched_pairs():
    rng = np.random.default_rng(3)
    A, B = [], []
    for _ in range(6):
        a, b = workloads.random_pair(rng, 300, 400, 4)
        A.append(a)
        B.append(b)
    got = L.lcs_batch(A, B)
    for a, b, r in zip(A, B, got):
        exp = O.lcs(a, b)
        assert (r.length, r.subsequence, r.row_positions, r.col_positions) == exp
    assert L.sweep_errors() == 0
