#!/usr/bin/env python3
"""Benchmark of the B200 Lu-Liu grid-graph LCS hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one exact LCS solve (leaf step -> every combine level -> recovery
walk -> assembly, results back on the host) of BASELINE.json config C
(default 5: m = n = 16384 over 26 letters, the largest config and the one the
roofline target is quoted on; configs 1-4 are parity cases, selectable here).
Inputs are seeded synthetic strings (workloads.py = SURVEY.md Appendix C); no
dataset exists for this path.

value  = m*n / device time per solve, strings already resident in HBM,
         CUDA events on the solve stream, L2 flushed (256 MiB write) between
         steps, max over ranks.
e2e    = same metric through the public API ``lcs(a, b)`` with HOST bytes in
         and LcsResult out (H2D of strings + plan, D2H of results timed).
roofline: dominant kernel = the combine levels (all heights: narrow levels,
         skeleton rows, row sweeps, finalize).  Algorithmic bytes per solve =
         8*OUT + 4*IN -- every output cell (reach + trace) written once, every
         input cell read once -- from the reference's own work counters
         (tests/golden/config_digests.json, counted by the C oracle), / the
         combine time measured live with CUDA events.  SURVEY.md 8(d)'s figure
         also charges 4*G for the gathers of the reference's per-row
         bisection; the row sweep no longer performs those, so that larger
         figure is reported beside it (`survey_8d`) but is not the fraction
         (it would exceed the bytes this code can possibly move).
cpu_baseline: the real reference (oracle/_ref, Cython backend) timed on this
         host on a bounded sample (leading sub-strings), else the C oracle port.

--impl reference runs the reference's own CPU path (oracle/_ref, all host
threads) on the same config's bounded sample; rank 0 only.
N > 1 (torchrun): ONE solve of the config split across the ranks (strong
scaling): each rank builds the reference tree's band subtrees, the upper
combines are sharded over start columns with NCCL broadcasts of finished row
ranges (paper_2309_09072_b200/distributed.py); --replicas runs
an independent instance per GPU instead (weak scaling).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "exact LCS cell-equivalents/sec (m*n/s)"
UNIT = "cells/s"
REF_SAMPLE = {1: 256, 2: 2048, 3: 2048, 4: 512, 5: 4096}  # leading-prefix length of the CPU sample


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--replicas", action="store_true",
                   help="N > 1: independent instance per GPU (weak) instead of one sharded solve")
    p.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of CPU baseline work")
    return p.parse_args()


def load_counters(cfg, seed):
    with open(os.path.join(ROOT, "tests", "golden", "config_digests.json")) as f:
        d = json.load(f)
    return d.get(f"cfg{cfg}/seed{seed}", {}).get("counters")


def load_digest(cfg, seed):
    with open(os.path.join(ROOT, "tests", "golden", "config_digests.json")) as f:
        return json.load(f).get(f"cfg{cfg}/seed{seed}")


def verify_timed_path(lib, _lib, build, m, n, swapped, digest):
    """One more solve of the exact timed path (traced build + device
    extraction), checked against the REFERENCE's digests of this config
    (tests/golden/config_digests.json, make_golden.py / make_deep_digests.py):
    LCS length, sha256 of subsequence and positions, of the final D_G and of
    the final trace table.  Outside the timed region."""
    import hashlib

    if digest is None:
        return "no reference digest for this config/seed"
    h = build()
    k = min(m, n)
    sub, rp, cp = np.empty(k, np.uint8), np.empty(k, np.int32), np.empty(k, np.int32)
    try:
        length = ctypes.c_int32()
        _lib.check(lib.lcsg_extract(h, -1, ctypes.byref(length), sub.ctypes.data, rp.ctypes.data,
                                    cp.ctypes.data), "extract")
        L = int(length.value)
        pa, pb = (cp[:L], rp[:L]) if swapped else (rp[:L], cp[:L])
        bad = []
        if L != digest["length"]:
            bad.append("length")
        if hashlib.sha256(sub[:L].tobytes()).hexdigest() != digest["subsequence_sha256"]:
            bad.append("subsequence")
        pos = np.concatenate([pa, pb]).astype(np.int64).tobytes()
        if hashlib.sha256(pos).hexdigest() != digest["positions_sha256"]:
            bad.append("positions")
        root = lib.lcsg_root(h)
        tab = np.empty((n + 1) * (min(m, n) + 1), np.int32)
        _lib.check(lib.lcsg_node_reach(h, root, tab.ctypes.data), "reach")
        if hashlib.sha256(tab.tobytes()).hexdigest() != digest["dg_sha256"]:
            bad.append("D_G")
        checked = "length, subsequence, positions, D_G"
        if "trace_sha256" in digest:
            _lib.check(lib.lcsg_node_trace(h, root, tab.ctypes.data), "trace")
            if hashlib.sha256(tab.tobytes()).hexdigest() != digest["trace_sha256"]:
                bad.append("trace")
            checked += ", trace"
    finally:
        lib.lcsg_free(h)
    return "ok" if not bad else "MISMATCH: " + ", ".join(bad) + f" (checked {checked})"


def load_cpu_full(cfg, seed):
    """The reference timed once on the WHOLE config (traced / low_memory, T=1 /
    all threads) on a GPU box's host by tools/cpu_full_baseline.py
    (profiles/cpu_full_cfgN.json); None if it was not run for this config."""
    path = os.path.join(ROOT, "profiles", f"cpu_full_cfg{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        doc = json.load(f)
    if doc.get("seed") != seed or not doc.get("best"):
        return None
    best = doc["best"]
    return {"value": best["cells_per_s"], "unit": UNIT, "cores": best["threads"],
            "kind": "reference", "seconds": best["seconds"], "mode": best["mode"],
            "cpu_model": doc["cpu_model"], "host_threads": doc["host_threads"],
            "runs": [{k: r.get(k) for k in ("mode", "threads", "seconds", "peak_rss_gb")}
                     for r in doc["runs"]],
            "source": f"profiles/cpu_full_cfg{cfg}.json (measured once, not in this run)"}


def load_issue(cfg):
    """Issue-slot utilisation of the dominant combine kernels from the
    committed ncu captures (profiles/issue_cfgN.json, tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", f"issue_cfg{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


def load_traffic(cfg):
    """DRAM bytes of one solve's combine launches from the committed ncu
    launch list (profiles/traffic_cfgN.json, tools/traffic.py); None if absent."""
    path = os.path.join(ROOT, "profiles", f"traffic_cfg{cfg}.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)["dram_bytes"]


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU legs (reference / oracle port): bounded samples
# ---------------------------------------------------------------------------
def cpu_impl():
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "lcsgrid_ref")):
        sys.path.insert(0, ref_dir)
        try:
            import lcsgrid_ref

            if lcsgrid_ref.active_backend() == "cython":
                return "reference", lambda a, b, t: lcsgrid_ref.lcs(a, b, threads=t).length
        except Exception:
            pass
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    return "port", lambda a, b, t: O.lcs(a, b, threads=t)[0]


def cpu_sample(cfg, seed):
    a, b = workloads.generate(cfg, seed)
    k = REF_SAMPLE[cfg]
    if cfg == 4:  # query x text: keep the query, take a text window
        return a[:k], b[: 64 * k]
    return a[:k], b[:k]


def cpu_baseline(cfg, seed, threads, budget_s):
    kind, fn = cpu_impl()
    a, b = cpu_sample(cfg, seed)
    times = []
    t_end = time.perf_counter() + budget_s
    while True:
        t0 = time.perf_counter()
        fn(a, b, threads)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end or len(times) >= 50:
            break
    t = statistics.median(times)
    return {"value": len(a) * len(b) / t, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"cfg{cfg} seed {seed} leading {len(a)}x{len(b)} sub-strings, "
                      f"median of {len(times)} solves ({t:.3f} s each)",
            "seconds_per_solve": t}


def run_reference(args, rank):
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    kind, fn = cpu_impl()
    a, b = cpu_sample(args.config, args.seed)
    for _ in range(args.warmup):
        fn(a, b, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        fn(a, b, threads)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    value = len(a) * len(b) / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": workloads.CONFIGS[args.config]["name"] + "_cpu_sample",
                   "m": len(a), "n": len(b), "seed": args.seed},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"cfg{args.config} leading {len(a)}x{len(b)} sub-strings"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU leg
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def run_ours(args, rank, world, dist):
    import torch

    from paper_2309_09072_b200 import _lib
    import paper_2309_09072_b200 as lcsgrid

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    seed = args.seed + rank
    a, b = workloads.generate(args.config, seed)
    rows, cols = (b, a) if len(a) > len(b) else (a, b)
    m, n = len(rows), len(cols)
    d_rows = torch.frombuffer(bytearray(rows), dtype=torch.uint8).to(dev)
    d_cols = torch.frombuffer(bytearray(cols), dtype=torch.uint8).to(dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    k = min(m, n)
    sub = np.empty(k, np.uint8)
    rp = np.empty(k, np.int32)
    cp = np.empty(k, np.int32)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > L2
    flags = _lib.LCSG_WITH_TRACE | _lib.LCSG_TIMING

    def build():
        h = ctypes.c_void_p()
        _lib.check(lib.lcsg_build_device(d_rows.data_ptr(), m, d_cols.data_ptr(), n, 1, m + 1,
                                         flags, local, sp, ctypes.byref(h)), "build")
        return h

    def solve():
        h = build()
        length = ctypes.c_int32()
        _lib.check(lib.lcsg_extract(h, -1, ctypes.byref(length), sub.ctypes.data,
                                    rp.ctypes.data, cp.ctypes.data), "extract")
        st = [ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double(),
              ctypes.c_int64(), ctypes.c_int64()]
        _lib.check(lib.lcsg_stats(h, *[ctypes.byref(x) for x in st]), "stats")
        lib.lcsg_free(h)
        return int(length.value), st[0].value, st[1].value, st[4].value, st[5].value

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize()
    step_ms, comb_ms, launches = [], [], 0
    h2d = d2h = 0
    length = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            length, nl, cms, h2d, d2h = solve()
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            comb_ms.append(cms)
            launches += nl
    t_ms = statistics.mean(step_ms)
    if dist is not None:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = world * m * n / (t_ms / 1e3)

    # e2e: public API, host bytes in / LcsResult out, same stream + events
    e2e_ms = []
    for it in range(max(2, min(args.steps, 5))):
        flush.zero_()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = lcsgrid.lcs(a, b, device=local, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if it > 0:  # first call is a warm-up of the host-input path
            e2e_ms.append(e0.elapsed_time(e1))
    assert r.length == length
    parity = verify_timed_path(lib, _lib, build, m, n, len(a) > len(b),
                               load_digest(args.config, seed))
    # the row-sweep kernels check the invariants they rely on: none may have failed
    sweep_bad = lcsgrid.sweep_errors(device=local)
    if sweep_bad:
        parity = f"row-sweep invariant violated {sweep_bad} times"
    e2e_t = statistics.mean(e2e_ms)
    if dist is not None:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_t = float(tt.item())

    if rank != 0:
        return
    peak, peak_kind = measured_peaks()
    counters = load_counters(args.config, seed)
    comb = statistics.mean(comb_ms)
    roof = None
    if counters:
        alg = 8 * counters["OUT"] + 4 * counters["IN"]
        alg_8d = 4 * counters["G"] + alg  # + the reference's Alg. 1 gathers
        achieved = alg / (comb / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": load_traffic(args.config),
                "traffic_source": "ncu dram__bytes_read+write of one solve's combine launches "
                                  f"(profiles/traffic_cfg{args.config}.json)",
                "kernel": "combine levels (all heights)", "combine_ms": comb,
                "algorithmic_bytes": alg, "peak_source": peak_kind,
                "bytes_per_cell": alg / (m * n),
                "survey_8d": {"algorithmic_bytes": alg_8d, "achieved": alg_8d / (comb / 1e3) / 1e9,
                              "frac": alg_8d / (comb / 1e3) / 1e9 / peak,
                              "note": "4*G + 8*OUT + 4*IN with the reference's gather count G; "
                                      "round 1's fraction (0.59) used this figure; the row sweep does not "
                                      "perform those gathers, so this can exceed 1"}}
        # INT32 term: C reference cell evaluations, one
        # 32-bit min each, at the IMNMX rate measured live on this GPU
        rate, sms, pms = ctypes.c_double(), ctypes.c_int32(), ctypes.c_double()
        if lib.lcsg_probe_int32_rate(local, ctypes.byref(rate), ctypes.byref(sms),
                                     ctypes.byref(pms)) == 0 and rate.value > 0:
            t_int = counters["C"] / rate.value * 1e3
            t_hbm = alg / (peak * 1e9) * 1e3
            roof["int32"] = {"rate_mins_per_s": rate.value, "sms": sms.value,
                             "ops": counters["C"], "t_roof_ms": t_int,
                             "frac": t_int / comb,
                             "source": "lcsg_probe_int32_rate: IMNMX.U32 chains, best of 5"}
            roof["t_roof_ms"] = max(t_hbm, t_int)
            roof["bound"] = "hbm" if t_hbm >= t_int else "int32"
        issue = load_issue(args.config)
        if issue:
            roof["issue_active"] = issue
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": workloads.CONFIGS[args.config]["name"], "m": m, "n": n,
                   "seed": args.seed, "lcs_length": length, "l2": "flushed (256 MiB) between steps",
                   "parallelism": f"replicas x{world}"},
        "roofline": roof,
        "parity": parity,
        "e2e": {"value": world * m * n / (e2e_t / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d + m + n), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args.config, args.seed, 1, args.cpu_budget)
        full = load_cpu_full(args.config, args.seed)
        if full is not None:
            line["cpu_baseline"]["full"] = full
    print(json.dumps(line), flush=True)


def run_sharded(args, rank, world, dist):
    """N > 1: ONE solve of the config split across the ranks (strong scaling):
    band subtrees per rank, upper combines sharded over start columns with
    NCCL broadcasts of finished row ranges (paper_2309_09072_b200.distributed)."""
    import torch

    from paper_2309_09072_b200 import distributed as D

    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    dev = torch.device("cuda", local)
    a, b = workloads.generate(args.config, args.seed)
    rows, cols = (b, a) if len(a) > len(b) else (a, b)
    m, n = len(rows), len(cols)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    r = None
    for _ in range(args.warmup):
        r = D.lcs_sharded(a, b, device=local)
    stats = D.CommStats()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = D.lcs_sharded(a, b, device=local, stats=stats)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    t_ms = statistics.mean(times)
    tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_ms = float(tt.item())
    # bytes each rank received through the schedule's collectives, per solve
    rb = torch.tensor([stats.received / max(1, args.steps)], dtype=torch.float64, device=dev)
    rb_all = [torch.zeros_like(rb) for _ in range(world)]
    dist.all_gather(rb_all, rb)
    received = [float(x.item()) for x in rb_all]
    _, bands, upper = D.build_plan(m, world)
    # kernels per solve on the busiest rank: its band build (~levels x 4) +
    # every upper combine (skeleton, 2 refinement stages, finalize)
    launches = args.steps * (4 * max(1, (m // max(1, len(bands))).bit_length()) + 4 * len(upper))
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": m * n / (t_ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": workloads.CONFIGS[args.config]["name"], "m": m, "n": n,
                   "seed": args.seed, "lcs_length": r.length,
                   "l2": "flushed (256 MiB) between steps",
                   "parallelism": f"{len(bands)} band subtrees + {len(upper)} upper combines "
                                  f"sharded over start columns across {world} GPUs (NCCL)"},
        "roofline": None,
        "comm": {"received_bytes_per_rank_per_solve": received,
                 "collectives": "2 all-gathers per upper combine (spans + kmax + wstar, then "
                                "finite-prefix reach rows) within each subtree's group; one "
                                "max all-reduce of the path"},
        "e2e": {"value": m * n / (t_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": m + n,
                "d2h_bytes_per_step": 4 * (m + 1)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
        # LCSG_DIST_BACKEND=gloo lets several ranks share one GPU for testing
        tdist.init_process_group(os.environ.get("LCSG_DIST_BACKEND", "nccl"))
        dist = tdist
    try:
        if world > 1 and not args.replicas:
            run_sharded(args, rank, world, dist)
        else:
            run_ours(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
