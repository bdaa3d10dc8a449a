"""Solve time on near-identical strings (worst case for the row sweep's register
capacity and walk lengths): b = a with a fraction of substitutions.
Usage: python tools/similar_strings.py [n] [fraction]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2309_09072_b200 as L

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
rng = np.random.default_rng(0)
A = rng.integers(0, 26, n) + 97
B = A.copy()
idx = rng.choice(n, int(frac * n), replace=False)
B[idx] = (B[idx] - 97 + rng.integers(1, 26, len(idx))) % 26 + 97
a, b = A.astype(np.uint8).tobytes(), B.astype(np.uint8).tobytes()
for env in ({}, {"LCSG_SWEEP": "0"}):
    for k, v in env.items():
        os.environ[k] = v
    L.sweep_paths(reset=True)
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = L.lcs(a, b)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"n={n} substitutions={frac}: {env or 'sweep'}: lcs {r.length}, "
          f"{1e3 * min(ts[1:]):.1f} ms per solve, sweep paths {L.sweep_paths()}, errors {L.sweep_errors()}")
    for k in env:
        del os.environ[k]
