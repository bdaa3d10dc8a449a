"""Seeded synthetic inputs of BASELINE.json's five configs.

No public dataset is involved: the reference ships no benchmark data, and
these generators (numpy PCG64, fixed draw order) are the stand-in the survey
defines.  Seed 0 is the headline; expected LCS lengths for seed 0 are
160 / 1782 / 1888 / 1024 / 5352.
"""

from __future__ import annotations

import numpy as np

ACGT = np.frombuffer(b"ACGT", dtype=np.uint8)

CONFIGS = {
    1: dict(name="cfg1_uniform4_256", m=256, n=256),
    2: dict(name="cfg2_mutated4_2048", m=2048, n=2048),
    3: dict(name="cfg3_dirichlet20_4096", m=4096, n=4096),
    4: dict(name="cfg4_query1024_text65536", m=1024, n=65536),
    5: dict(name="cfg5_uniform26_16384", m=16384, n=16384),
}
EXPECTED_LCS_SEED0 = {1: 160, 2: 1782, 3: 1888, 4: 1024, 5: 5352}


def generate(cfg: int, seed: int = 0):
    """Return (a, b) as bytes for config ``cfg`` (1..5)."""
    rng = np.random.default_rng(seed)
    if cfg == 1:
        A = rng.integers(0, 4, 256)
        B = rng.integers(0, 4, 256)
        return ACGT[A].tobytes(), ACGT[B].tobytes()
    if cfg == 2:
        A = rng.integers(0, 4, 2048)
        B = A.copy()
        for p in rng.choice(2048, 204, replace=False):
            B[p] = (B[p] + rng.integers(1, 4)) % 4
        dels = set(int(x) for x in rng.choice(2048, 102, replace=False))
        B = [int(v) for q, v in enumerate(B) if q not in dels]
        for _ in range(102):
            p = int(rng.integers(0, len(B) + 1))
            B.insert(p, int(rng.integers(0, 4)))
        return ACGT[A].tobytes(), ACGT[np.array(B)].tobytes()
    if cfg == 3:
        p = rng.dirichlet(np.ones(20))
        A = rng.choice(20, 4096, p=p)
        B = rng.choice(20, 4096, p=p)
        return (A + 65).astype(np.uint8).tobytes(), (B + 65).astype(np.uint8).tobytes()
    if cfg == 4:
        Q = rng.integers(0, 4, 1024)
        T = rng.integers(0, 4, 65536)
        offs = sorted(int(x) for x in rng.choice(65536 - 1024, 8, replace=False))
        for o in offs:
            q = Q.copy()
            idx = rng.choice(1024, 51, replace=False)
            q[idx] = (q[idx] + rng.integers(1, 4, 51)) % 4
            T[o:o + 1024] = q
        return ACGT[Q].tobytes(), ACGT[T].tobytes()
    if cfg == 5:
        A = rng.integers(0, 26, 16384) + 97
        B = rng.integers(0, 26, 16384) + 97
        return A.astype(np.uint8).tobytes(), B.astype(np.uint8).tobytes()
    raise ValueError(f"unknown config {cfg}")


def cfg4_planted_windows(seed: int = 0, width: int = 8192):
    """Batched-solve workload: cfg4's query against a
    text window of ``width`` columns around each of its 8 planted copies --
    8 equal-shape pairs (1024 x width).  The planted offsets are re-drawn
    exactly as generate(4, seed) draws them."""
    a, b = generate(4, seed)
    rng = np.random.default_rng(seed)
    rng.integers(0, 4, 1024)
    rng.integers(0, 4, 65536)
    offs = sorted(int(x) for x in rng.choice(65536 - 1024, 8, replace=False))
    pairs = []
    for o in offs:
        lo = min(max(0, o + 512 - width // 2), len(b) - width)
        pairs.append((a, b[lo:lo + width]))
    return pairs


def random_pair(rng, m: int, n: int, sigma: int, base: int = 97):
    """Small i.i.d. uniform test pair (used by the parity sweeps)."""
    a = (rng.integers(0, sigma, m) + base).astype(np.uint8).tobytes()
    b = (rng.integers(0, sigma, n) + base).astype(np.uint8).tobytes()
    return a, b
