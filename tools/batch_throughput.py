"""Throughput of many small solves: sequential lcs() vs lcs_many()."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_09072_b200 as L
import workloads

rng = np.random.default_rng(0)
for size, count in ((256, 64), (1024, 32), (2048, 16)):
    pairs = [workloads.random_pair(rng, size, size, 4) for _ in range(count)]
    L.lcs_many(pairs[:4])
    t0 = time.perf_counter(); seq = [L.lcs(a, b) for a, b in pairs]; t1 = time.perf_counter()
    for c in (4, 8, 16):
        t2 = time.perf_counter(); par = L.lcs_many(pairs, concurrency=c); t3 = time.perf_counter()
        assert par == seq
        print(f"{count} x {size}^2: sequential {1e3*(t1-t0)/count:.3f} ms/pair, "
              f"lcs_many(concurrency={c}) {1e3*(t3-t2)/count:.3f} ms/pair")
