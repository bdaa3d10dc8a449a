"""Randomised parity sweep on the GPU against the C oracle (test infrastructure):
lcs() outputs and the final D_G of random pairs over a range of shapes,
alphabets and orientations (m > n included), until a time budget runs out.
Usage: python tools/fuzz_parity.py [seconds] [seed]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import oracle as O
import paper_2309_09072_b200 as L
import workloads

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
t_end = time.time() + budget
n_cases = 0
shapes = [(1, 1), (1, 50), (50, 1), (7, 3000), (2, 9000), (130, 130), (257, 300), (600, 700),
          (1100, 900), (300, 9500), (64, 20000), (1500, 1600), (2100, 2100)]
while time.time() < t_end:
    m0, n0 = shapes[n_cases % len(shapes)]
    m = max(1, int(m0 * rng.uniform(0.7, 1.3)))
    n = max(1, int(n0 * rng.uniform(0.7, 1.3)))
    sigma = int(rng.choice([2, 4, 20, 26, 200]))
    a, b = workloads.random_pair(rng, m, n, sigma)
    if rng.random() < 0.3:  # planted similarity: long LCS
        k = min(len(a), len(b))
        bb = bytearray(b)
        src = np.frombuffer(a, np.uint8)[:k]
        mask = rng.random(k) < 0.8
        arr = np.frombuffer(bytes(bb), np.uint8).copy()
        arr[:k][mask] = src[mask]
        b = arr.tobytes()
    low = bool(rng.random() < 0.25)
    got = L.lcs(a, b, low_memory=low)
    exp = O.lcs(a, b)
    assert (got.length, got.subsequence, got.row_positions, got.col_positions) == exp, \
        f"lcs mismatch m={m} n={n} sigma={sigma} low={low}"
    if m <= n and m * n <= 4_000_000:
        g = L.GridModel(a, b)
        tab = L.build_cost_table(g, 1, g.m + 1, with_trace=not low)
        t = O.OracleTree(a, b)
        assert np.array_equal(tab.reach, t.node(t.root).reach), f"D_G mismatch m={m} n={n}"
    n_cases += 1
print(f"fuzz ok: {n_cases} random cases bit-exact vs the oracle")
