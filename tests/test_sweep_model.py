"""The row-sweep recurrence (tests/sweep_model.py) regenerates
every row of every combine of the oracle's trees -- reach and first-wins
traces of the finite cells, kmax, the insertion ranks -- from the row above.
CPU only: pins the structure the CUDA sweep kernels rely on."""

import numpy as np
import pytest

import oracle as O
import sweep_model
import workloads


def _check_tree(a, b, stride=None, min_rows=2):
    t = O.OracleTree(a, b)
    stats = {}
    for idx in range(len(t)):
        nd = t.node(idx)
        if nd.upper < 0 or nd.bottom_row - nd.top_row < min_rows:
            continue
        sweep_model.sweep_node(nd, t.node(nd.upper), t.node(nd.lower), t.inf, stride, stats)
    return stats


@pytest.mark.parametrize("sigma", [2, 4, 26])
def test_recurrence_random(sigma):
    rng = np.random.default_rng(sigma)
    for _ in range(3):
        m, n = int(rng.integers(20, 70)), int(rng.integers(10, 90))
        a, b = workloads.random_pair(rng, m, n, sigma)
        st = _check_tree(a, b)
        assert st["rows"] > 0


def test_recurrence_structured_and_strided():
    cases = [(b"a" * 40, b"a" * 55), (b"abc" * 15, b"x" * 30), (b"ab" * 25, b"ba" * 30),
             (b"gatttatgcagg", b"tcaggatt"), (b"tcaggatt", b"gatttatgcagg")]
    for a, b in cases:
        _check_tree(a, b)
        _check_tree(a, b, stride=4)


def test_recurrence_planted_copy_long_walks():
    rng = np.random.default_rng(8)
    a, b = workloads.random_pair(rng, 90, 110, 200)
    arr = np.frombuffer(b, np.uint8).copy()
    src = np.frombuffer(a, np.uint8)
    mask = rng.random(90) < 0.8
    arr[:90][mask] = src[mask]
    st = _check_tree(a, arr.tobytes(), min_rows=16)
    assert st["walk"] / st["rows"] > 1.0  # walks longer than the inserted cell alone
