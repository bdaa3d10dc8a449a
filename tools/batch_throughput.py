"""Throughput of many small solves: sequential lcs()
vs independent solves on concurrent streams (lcs_many(batch=False)) vs ONE
batched solve per shape (lcs_batch: one launch per tree height for all
pairs).  Wall clock per pair, host strings in / LcsResult out, after a
warm-up of each path; every result checked against the sequential one.

    python tools/batch_throughput.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2309_09072_b200 as L  # noqa: E402
import workloads  # noqa: E402


def timed(fn, reps=3):
    fn()  # warm-up (arena pool, layout cache)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        dt = time.perf_counter() - t0
        best = dt if best is None or dt < best else best
    return best, r


rng = np.random.default_rng(0)
cases = [("cfg4 query x 8 planted windows (1024 x 8192)", workloads.cfg4_planted_windows(0, 8192))]
for size, count in ((256, 64), (1024, 32), (2048, 16)):
    cases.append((f"{count} x {size}^2 sigma=4",
                  [workloads.random_pair(rng, size, size, 4) for _ in range(count)]))
rows = []
for name, pairs in cases:
    A = [a for a, _ in pairs]
    B = [b for _, b in pairs]
    t_seq, seq = timed(lambda: [L.lcs(a, b) for a, b in pairs])
    t_str, par = timed(lambda: L.lcs_many(pairs, batch=False, concurrency=8))
    t_bat, bat = timed(lambda: L.lcs_batch(A, B))
    assert par == seq and bat == seq, name
    cells = sum(len(a) * len(b) for a, b in pairs)
    row = {"workload": name, "pairs": len(pairs),
           "ms_per_pair": {"sequential": 1e3 * t_seq / len(pairs),
                           "streams_x8": 1e3 * t_str / len(pairs),
                           "batched": 1e3 * t_bat / len(pairs)},
           "cells_per_s": {"sequential": cells / t_seq, "streams_x8": cells / t_str,
                           "batched": cells / t_bat},
           "speedup_batched_vs_sequential": t_seq / t_bat}
    rows.append(row)
    print(json.dumps(row), flush=True)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(rows, f, indent=1)
