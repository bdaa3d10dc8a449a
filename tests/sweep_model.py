"""Executable statement of the row-sweep recurrence in plain
Python / numpy -- TEST INFRASTRUCTURE: tests/test_sweep_model.py runs it on
the CPU against the oracle's tables, so the recurrence the CUDA sweep kernels
(paper_2309_09072_b200/csrc/lcsg_sweep.cu) implement is pinned without a GPU.

Given the children tables U, L and ONE finished row c of the combine
C = U (x) L (solver.py:91-110, _kernel.pyx:14-82), `next_row` produces row
c + 1 -- reach values and first-wins splits -- touching only the few cells
between the insertion rank j1 and J.
"""

import numpy as np


def event_rank(row_next, row_cur, inf):
    """Insertion rank of row c+1 against row c: first k with
    row_next[k] != row_cur[k+1] (len(row) when nothing was inserted)."""
    shifted = np.concatenate([row_cur[1:], [inf]])
    neq = np.nonzero(row_next != shifted)[0]
    return int(neq[0]) if len(neq) else len(row_next)


def next_row(R, T, K, U_next, kmax_u_next, ju1, L, inf, stats=None):
    """Row c+1 of the combine from row c = (R, T, K): R reach values, T
    first-wins splits, K last finite index.  U_next = U[c+1], ju1 = U's event
    rank from row c to c+1, L the lower table.  Returns (R', T', K', j1)."""
    w1 = len(R)
    wl = L.shape[1] - 1
    newR = np.full(w1, inf, np.int64)
    newT = np.zeros(w1, np.int64)

    def cell(j, klo, khi):  # first-wins minimum over the splits [klo, khi]
        best = (inf, 0)
        for k in range(klo, khi + 1):
            x = int(U_next[k])
            v = int(L[x - 1][j - k]) if (x < inf and j - k <= wl) else inf
            if stats is not None:
                stats["gathers"] = stats.get("gathers", 0) + 1
            if v < best[0]:
                best = (v, k)
        return best

    # J: last cell whose split lies left of U's insertion (splits are nondecreasing)
    J = max(j for j in range(K + 1) if T[j] <= ju1)
    assert all(T[j] <= ju1 for j in range(J + 1)), "splits not monotone"
    newR[J + 1:K + 1] = R[J + 1:K + 1]  # unchanged cells
    newT[J + 1:K + 1] = T[J + 1:K + 1]
    j1 = None
    for j in range(J, -1, -1):  # the walk
        ub = min(j, kmax_u_next)
        if j == J:
            if J < K:
                ub = min(ub, int(T[J + 1]))
        else:
            ub = min(ub, int(newT[j + 1]))
        klo = max(ju1, j - wl, 0)
        v, k = cell(j, klo, ub) if klo <= ub else (inf, 0)
        if v == R[j] and v < inf:  # value kept, split moved right of U's insertion
            newR[j], newT[j] = v, k
            continue
        j1 = j  # the inserted cell (INF: nothing inserted, the row gets shorter)
        if v < inf:
            newR[j], newT[j] = v, k
        break
    assert j1 is not None, "cell 0 always changes"
    Kn = K if newR[j1] < inf else K - 1
    if newR[j1] >= inf:
        assert j1 == K
    for j in range(j1):  # shifted cells; a zero split stays zero
        newR[j] = R[j + 1]
        newT[j] = max(int(T[j + 1]) - 1, 0)
    if stats is not None:
        stats["rows"] = stats.get("rows", 0) + 1
        stats["walk"] = stats.get("walk", 0) + (J - j1 + 1)
    return newR, newT, Kn, j1


def sweep_node(C, U, L, inf, stride=None, stats=None):
    """Regenerate every row of combine node C from its first row (or from
    every `stride`-th row, like the kernels' skeleton) and compare with C."""
    n1, w1 = C.reach.shape
    R = T = K = None
    for c in range(n1 - 1):
        if R is None or (stride and c % stride == 0):
            R, T, K = C.reach[c].astype(np.int64), C.trace[c].astype(np.int64), int(C.kmax[c])
        ju1 = event_rank(U.reach[c + 1], U.reach[c], inf)
        R, T, K, j1 = next_row(R, T, K, U.reach[c + 1], int(U.kmax[c + 1]), ju1, L.reach, inf, stats)
        exp_k = int(C.kmax[c + 1])
        assert K == exp_k, (c, K, exp_k)
        assert np.array_equal(R[:K + 1], C.reach[c + 1][:K + 1]), ("reach", c)
        assert np.all(C.reach[c + 1][K + 1:] >= inf)
        assert np.array_equal(T[:K + 1], C.trace[c + 1][:K + 1]), ("trace", c)
        assert j1 == event_rank(C.reach[c + 1], C.reach[c], inf) or C.reach[c + 1][j1] >= inf
