"""Quadratic DP LCS with deterministic backtrack (reference oracle.py:15-63).

Part of the reference package's public API (``lcsgrid.dp_lcs``), re-provided
here for drop-in completeness; it is a differential checker, not the hot
path.  Row updates are vectorised: for a match row the LCS recurrence
cur[j] = max(prev[j], cur[j-1], prev[j-1]+1 if match) equals a running
maximum of max(prev[j], match*(prev[j-1]+1)).
"""

from __future__ import annotations

import numpy as np

from .seqcore import LcsResult, SequenceLike, as_bytes


def dp_table(a: SequenceLike, b: SequenceLike) -> list:
    """(m+1) x (n+1) LCS-length table as nested lists (reference oracle.py:15-33)."""
    return _table(as_bytes(a), as_bytes(b)).tolist()


def _table(aa: bytes, bb: bytes) -> np.ndarray:
    m, n = len(aa), len(bb)
    T = np.zeros((m + 1, n + 1), dtype=np.int32)
    cols = np.frombuffer(bb, dtype=np.uint8)
    for i, ca in enumerate(aa, start=1):
        prev = T[i - 1]
        cand = prev[1:].copy()
        hit = cols == ca
        cand[hit] = np.maximum(cand[hit], prev[:-1][hit] + 1)
        T[i, 1:] = np.maximum.accumulate(cand)
    return T


def dp_lcs(a: SequenceLike, b: SequenceLike) -> LcsResult:
    """Exact LCS by DP; backtrack prefers diagonal, then up, then left
    (reference oracle.py:36-63)."""
    aa, bb = as_bytes(a), as_bytes(b)
    T = _table(aa, bb)
    i, j = len(aa), len(bb)
    picked = []
    while i > 0 and j > 0:
        if aa[i - 1] == bb[j - 1]:
            picked.append((i, j))
            i -= 1
            j -= 1
        elif T[i - 1, j] >= T[i, j - 1]:
            i -= 1
        else:
            j -= 1
    picked.reverse()
    return LcsResult(
        length=len(picked),
        subsequence=bytes(aa[p - 1] for p, _ in picked),
        row_positions=tuple(p for p, _ in picked),
        col_positions=tuple(q for _, q in picked),
    )
