"""Latency of a process's first solves: wall time of
lcs() for the first cfg1 solve (library / module loading), the first cfg5
solve (arena pool growth), and a repeated cfg5 solve, with the host phase
split from LCSG_HOST_PROFILE=1 on stderr.
    python tools/first_solve.py [--reserve GB]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_09072_b200 as L
import workloads

reserve = float(sys.argv[sys.argv.index("--reserve") + 1]) if "--reserve" in sys.argv else 0.0
if reserve:
    t0 = time.perf_counter()
    L.reserve(int(reserve * 2**30))
    print(f"reserve {reserve} GB: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
for name, cfg in (("cfg1 first", 1), ("cfg1 again", 1), ("cfg5 first", 5), ("cfg5 again", 5),
                  ("cfg5 third", 5)):
    a, b = workloads.generate(cfg)
    t0 = time.perf_counter()
    r = L.lcs(a, b)
    print(f"{name}: {1e3 * (time.perf_counter() - t0):.1f} ms (length {r.length})", flush=True)
