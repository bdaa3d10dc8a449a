"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), checked against the C oracle so a run also proves the result:

    compute-sanitizer --tool memcheck  python tools/sanitize_case.py
    compute-sanitizer --tool racecheck python tools/sanitize_case.py

Cases: cfg1 (256 x 256, traced and low-memory), a 300 x 420 sigma=4 pair
(wide tables: skeleton + column refinement + finalize), a 64 x 6000
sigma=256 pair (narrow kernels' direct-read path past the staged L window),
each also with forced 64-bit keys (LCSG_FORCE_KEY64=1).
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2309_09072_b200 as L  # noqa: E402
import workloads  # noqa: E402


def cases():
    rng = np.random.default_rng(5150)
    yield "cfg1", workloads.generate(1)
    yield "300x420", workloads.random_pair(rng, 300, 420, 4)
    a = rng.integers(0, 256, 64).astype(np.uint8).tobytes()
    b = rng.integers(0, 256, 6000).astype(np.uint8).tobytes()
    yield "64x6000", (a, b)


def main():
    which = sys.argv[1:] or ["0", "1"]
    for key64 in which:
        os.environ["LCSG_FORCE_KEY64"] = key64
        for name, (a, b) in cases():
            exp = O.lcs(a, b)
            for low in (False, True):
                r = L.lcs(a, b, low_memory=low)
                got = (r.length, r.subsequence, r.row_positions, r.col_positions)
                assert got == exp, (name, key64, low)
            g = L.GridModel(a, b)
            tab = L.build_cost_table(g, 1, g.m + 1)
            t = O.OracleTree(a, b)
            np.testing.assert_array_equal(tab.reach, t.node(t.root).reach)
            np.testing.assert_array_equal(tab.trace, t.node(t.root).trace)
            print(f"ok {name} key64={key64}", flush=True)


if __name__ == "__main__":
    main()
