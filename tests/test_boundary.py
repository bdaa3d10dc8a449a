"""The drop-in boundary exercised from the REFERENCE side.

* The kernel-level plugin (paper_2309_09072_b200/reference_plugin.py) is
  registered as ``lcsgrid_ref._backend.BACKENDS["cuda"]`` of the unmodified
  reference build (oracle/_ref) and the reference's own ``build_cost_table``
  / ``lcs`` run through it: every node and every result must equal the
  reference's Cython backend bit for bit (reference _backend.py:20-22,40-50,
  _kernel.pyx:63-82).
* The public ``combine_row`` (reference solver.py:142-157) against the
  reference's on reference trees.
"""

import numpy as np
import pytest

import paper_2309_09072_b200 as L
import workloads
from paper_2309_09072_b200 import reference_plugin


def _nodes(table):
    out = []

    def rec(t):
        if t.upper is not None:
            rec(t.upper)
            rec(t.lower)
        out.append(t)

    rec(table)
    return out


def test_plugin_rejects_bad_buffers():
    """Reference contract: wrong dtype / non-contiguous buffers raise
    ValueError at the call (Cython typed memoryviews, _kernel.pyx:63-66)."""
    u = np.zeros((4, 3), np.intc)
    k = np.zeros(4, np.intc)
    with pytest.raises(ValueError, match="int32"):
        reference_plugin.combine_level(u.astype(np.int64), k, u, 1, u, u, True, 9, 0, 4)
    with pytest.raises(ValueError, match="C-contiguous"):
        reference_plugin.combine_level(np.asfortranarray(np.zeros((4, 3), np.intc)), k, u, 1, u,
                                       u, True, 9, 0, 4)
    assert reference_plugin.NAME == "cuda"


@pytest.fixture
def ref_with_cuda(reference):
    from lcsgrid_ref import _backend as B

    B.BACKENDS["cuda"] = reference_plugin
    yield reference
    B.BACKENDS.pop("cuda", None)


@pytest.mark.gpu
def test_reference_solver_through_cuda_plugin(ref_with_cuda):
    R = ref_with_cuda
    from lcsgrid_ref import seqcore as Rs, solver as Rv

    rng = np.random.default_rng(31)
    cases = [(b"tcaggatt", b"gatttatgcagg")]
    cases += [workloads.random_pair(rng, int(rng.integers(1, 120)), int(rng.integers(0, 300)),
                                    int(rng.choice([2, 4, 26]))) for _ in range(16)]
    cases.append(workloads.generate(1))
    for a, b in cases:
        g = Rs.GridModel(a, b)
        for with_trace in (True, False):
            for threads in (1, 3):
                got = Rv.build_cost_table(g, 1, g.m + 1, backend="cuda", threads=threads,
                                          with_trace=with_trace)
                exp = Rv.build_cost_table(g, 1, g.m + 1, backend="cython", with_trace=with_trace)
                for x, y in zip(_nodes(got), _nodes(exp), strict=True):
                    np.testing.assert_array_equal(x.reach, y.reach)
                    np.testing.assert_array_equal(x.kmax, y.kmax)
                    assert x.wstar == y.wstar
                    if with_trace and y.trace is not None:
                        np.testing.assert_array_equal(x.trace, y.trace)
        for low in (False, True):
            assert R.lcs(a, b, backend="cuda", low_memory=low) == R.lcs(a, b, backend="cython")


@pytest.mark.gpu
def test_combine_row_matches_reference(reference):
    from lcsgrid_ref import seqcore as Rs, solver as Rv

    rng = np.random.default_rng(32)
    for _ in range(8):
        m, n = int(rng.integers(2, 90)), int(rng.integers(1, 200))
        a, b = workloads.random_pair(rng, m, n, int(rng.choice([2, 4, 26])))
        ours = L.build_cost_table(L.GridModel(a, b), 1, m + 1)
        ref = Rv.build_cost_table(Rs.GridModel(a, b), 1, m + 1)
        for i in sorted({1, n + 1, *(int(x) for x in rng.integers(1, n + 2, 5))}):
            row, tr = L.combine_row(ours.upper.row(i), ours.lower, ours.max_weight)
            erow, etr = Rv.combine_row(ref.upper.row(i), ref.lower, ref.max_weight)
            assert row.start == erow.start == i
            np.testing.assert_array_equal(row.reach, erow.reach)
            np.testing.assert_array_equal(tr, etr)
            np.testing.assert_array_equal(row.reach, ref.reach[i - 1])
