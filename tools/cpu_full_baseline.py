"""Full-config CPU baseline of the REFERENCE.

    python tools/cpu_full_baseline.py [--config 5] [--out profiles/cpu_full_cfg5.json]

Times the unmodified reference ``lcsgrid_ref.lcs(a, b, threads=T)``
(oracle/_ref, Cython backend) on the WHOLE config (no sample), traced and
``low_memory=True``, at T=1 and T=all host threads, each run in a fresh
subprocess (peak RSS measured per run), and records the host CPU model.
Run it once on the GPU box; bench.py reports the file as cpu_baseline.full.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import resource
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, time, resource
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "oracle", "_ref"))
import workloads, lcsgrid_ref
assert lcsgrid_ref.active_backend() == "cython"
a, b = workloads.generate({cfg}, {seed})
t0 = time.perf_counter()
r = lcsgrid_ref.lcs(a, b, threads={threads}, low_memory={low})
dt = time.perf_counter() - t0
print(json.dumps({{"seconds": dt, "length": r.length,
                  "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20}}))
"""


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", type=int, default=5)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--threads", default="1,all")
    p.add_argument("--modes", default="traced,low_memory")
    p.add_argument("--out", default=None)
    args = p.parse_args()
    allt = len(os.sched_getaffinity(0))
    threads = [allt if t == "all" else int(t) for t in args.threads.split(",")]
    import workloads

    a, b = workloads.generate(args.config, args.seed)
    runs = []
    for mode in args.modes.split(","):
        for t in threads:
            code = CHILD.format(root=ROOT, cfg=args.config, seed=args.seed, threads=t,
                                low=(mode == "low_memory"))
            t0 = time.time()
            res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
            if res.returncode != 0:
                runs.append({"mode": mode, "threads": t, "error": res.stderr[-400:]})
                continue
            out = json.loads(res.stdout.strip().splitlines()[-1])
            out.update({"mode": mode, "threads": t, "wall_incl_startup": time.time() - t0,
                        "cells_per_s": len(a) * len(b) / out["seconds"]})
            runs.append(out)
            print(json.dumps(out), flush=True)
    ok = [r for r in runs if "seconds" in r]
    best = min(ok, key=lambda r: r["seconds"]) if ok else None
    doc = {"config": args.config, "seed": args.seed, "m": len(a), "n": len(b),
           "cpu_model": cpu_model(), "host_threads": allt,
           "impl": "reference lcsgrid_ref.lcs (oracle/_ref, Cython backend), full config",
           "runs": runs, "best": best}
    out = args.out or os.path.join(ROOT, "profiles", f"cpu_full_cfg{args.config}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({"best": best, "cpu_model": doc["cpu_model"], "host_threads": allt}))


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    main()
