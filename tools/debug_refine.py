"""Debug helper (not part of the product): hunt refinement parity failures.

    python tools/debug_refine.py ITER [ENV=VAL ...]

Runs ITER random instances (sizes/alphabets like tests/test_gpu_parity.py)
under the given LCSG_* environment and prints the first mismatching node with
its bad cells, compared with the C oracle.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
import paper_2309_09072_b200 as L  # noqa: E402
import workloads  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    os.environ[k] = v
rng = np.random.default_rng(12345)


def nodes_of(tab):
    out = []

    def rec(x):
        if x.upper is not None:
            rec(x.upper)
            rec(x.lower)
        out.append(x)

    rec(tab)
    return out


for it in range(iters):
    m = int(rng.integers(4, 330))
    n = int(rng.integers(2, 420))
    sigma = int(rng.choice([2, 3, 4, 20, 26]))
    a, b = workloads.random_pair(rng, m, n, sigma)
    g = L.GridModel(a, b)
    t = O.OracleTree(a, b)
    nodes = nodes_of(L.build_cost_table(g, 1, m + 1))
    for idx in range(len(t)):
        e = t.node(idx)
        if e.upper < 0:
            continue
        got = nodes[idx]
        for name, gv, ev in (("reach", got.reach, e.reach), ("trace", got.trace, e.trace),
                             ("kmax", got.kmax[:, None], e.kmax[:, None])):
            bad = np.argwhere(gv != ev)
            if len(bad):
                U = t.node(e.upper)
                print(f"it={it} m={m} n={n} sigma={sigma} node={idx} rows {e.top_row}..{e.bottom_row} "
                      f"w1={e.reach.shape[1]} {name} bad={len(bad)} wstarL={t.node(e.lower).wstar}")
                for r, c in bad[:12]:
                    print(f"  ({r},{c}) got {gv[r, c]} want {ev[r, c]}  reach_want={e.reach[r, c]} "
                          f"trace_want={e.trace[r, c]} kmax={e.kmax[r]} kmaxU={U.kmax[r]}")
                r0 = int(bad[0][0]); c0 = int(bad[0][1])
                lo, hi = (r0 // 16) * 16, min((r0 // 16) * 16 + 16, e.reach.shape[0] - 1)
                print("  rows", lo, "..", hi, "col", c0)
                print("  want", [int(x) for x in e.reach[lo:hi + 1, c0]])
                print("  got ", [int(x) for x in got.reach[lo:hi + 1, c0]])
                print("  kmaxU", [int(x) for x in U.kmax[lo:hi + 1]])
                print("  kmax ", [int(x) for x in e.kmax[lo:hi + 1]])
                sys.exit(1)
print("no mismatch in", iters, "instances")
