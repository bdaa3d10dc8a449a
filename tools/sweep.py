"""Schedule sweep: combine time of one config under several env settings, in
one process (the library reads its LCSG_* knobs at every build).
Usage: python tools/sweep.py CFG [--reps R] [--levels] "K=V,K2=V2" "K=V" ...
("" = defaults).  --levels prints the per-launch kernel durations of one
solve per setting (CUPTI via torch.profiler; not a bench number)."""
import argparse, ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_09072_b200 import _lib
import workloads

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("settings", nargs="*")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--levels", action="store_true")
ap.add_argument("--lowmem", action="store_true", help="build without stored traces")
args = ap.parse_intermixed_args()
lib = _lib.load()
a, b = workloads.generate(args.cfg)
rows, cols = (b, a) if len(a) > len(b) else (a, b)
m, n = len(rows), len(cols)
dev = torch.device("cuda", 0)
d_rows = torch.frombuffer(bytearray(rows), dtype=torch.uint8).to(dev)
d_cols = torch.frombuffer(bytearray(cols), dtype=torch.uint8).to(dev)
s = torch.cuda.current_stream()
sp = ctypes.c_void_p(s.cuda_stream)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
k = min(m, n)
sub = np.empty(k, np.uint8); rp = np.empty(k, np.int32); cp = np.empty(k, np.int32)


def solve():
    h = ctypes.c_void_p()
    _lib.check(lib.lcsg_build_device(d_rows.data_ptr(), m, d_cols.data_ptr(), n, 1, m + 1,
                                     (0 if args.lowmem else _lib.LCSG_WITH_TRACE) | _lib.LCSG_TIMING, 0, sp,
                                     ctypes.byref(h)), "build")
    length = ctypes.c_int32()
    _lib.check(lib.lcsg_extract(h, -1, ctypes.byref(length), sub.ctypes.data, rp.ctypes.data,
                                cp.ctypes.data), "extract")
    st = [ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double(),
          ctypes.c_int64(), ctypes.c_int64()]
    _lib.check(lib.lcsg_stats(h, *[ctypes.byref(x) for x in st]), "stats")
    lib.lcsg_free(h)
    return length.value, st[1].value


def clocks():
    import subprocess
    q = "clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw"
    r = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"],
                       capture_output=True, text=True)
    return r.stdout.strip()


print("# clocks before:", clocks(), flush=True)
base_env = {k2: v for k2, v in os.environ.items() if k2.startswith("LCSG_")}
ref_len = None
for setting in [("" if x == "default" else x) for x in (args.settings or ["default"])]:
    for k2 in [x for x in os.environ if x.startswith("LCSG_")]:
        del os.environ[k2]
    os.environ.update(base_env)
    for kv in filter(None, setting.split(",")):
        k2, v = kv.split("=")
        os.environ[k2] = v
    solve()
    ts = []
    for _ in range(args.reps):
        flush.zero_()
        torch.cuda.synchronize()
        ln, cms = solve()
        ts.append(cms)
    ref_len = ref_len if ref_len is not None else ln
    ok = "" if ln == ref_len else f"  LENGTH MISMATCH {ln} vs {ref_len}"
    print(f"{setting or 'default':60s} combine {statistics.median(ts):8.3f} ms "
          f"(min {min(ts):.3f}){ok}", flush=True)
    print("#   clocks:", clocks(), flush=True)
    if args.levels:
        from torch.profiler import profile, ProfilerActivity
        flush.zero_(); torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            solve()
            torch.cuda.synchronize()
        evs = [e for e in prof.events() if e.device_type.name == "CUDA" and "kernel" in e.name.lower()
               or (e.device_type.name == "CUDA" and not e.name.startswith("Memcpy")
                   and not e.name.startswith("Memset"))]
        for e in evs:
            print(f"   {e.name.split('(')[0][:60]:60s} {e.device_time:9.1f} us")
