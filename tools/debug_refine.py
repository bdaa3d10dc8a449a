"""Debug helper: reproduce a refinement parity failure and print the bad cells."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O
import paper_2309_09072_b200 as L
import workloads

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 64
os.environ["LCSG_SKELETON_STRIDE"] = str(stride)
rng = np.random.default_rng(100 + stride)
for it in range(12):
    m = int(rng.integers(66, 330)); n = int(rng.integers(40, 420)); sigma = int(rng.choice([2, 4, 20, 26]))
    a, b = workloads.random_pair(rng, m, n, sigma)
    g = L.GridModel(a, b)
    t = O.OracleTree(a, b)
    for with_trace in (True, False):
        tab = L.build_cost_table(g, 1, m + 1, with_trace=with_trace)
        nodes = []
        def rec(x):
            if x.upper is not None:
                rec(x.upper); rec(x.lower)
            nodes.append(x)
        rec(tab)
        for idx in range(len(t)):
            e = t.node(idx)
            if e.upper < 0:
                continue
            gr = nodes[idx].reach
            bad = np.argwhere(gr != e.reach)
            if len(bad):
                print(f"it={it} m={m} n={n} sigma={sigma} trace={with_trace} node={idx} rows {e.top_row}..{e.bottom_row} w1={gr.shape[1]} bad={len(bad)}")
                rows = sorted(set(int(r) for r, _ in bad))
                print("bad rows", rows[:40])
                for r, c in bad[:12]:
                    print(f"  cell ({r},{c}) got {gr[r,c]} want {e.reach[r,c]} trace_want {e.trace[r,c]} kmax_want {e.kmax[r]} kmax_got {nodes[idx].kmax[r]}")
                sys.exit(0)
print("no mismatch")
