"""Per-level statistics of the row-sweep kernel (needs a library built with
-DLCSG_SWEEP_STATS: LCSG_NVCC_EXTRA=-DLCSG_SWEEP_STATS python tools/sweep_stats.py 5)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2309_09072_b200 as L
from paper_2309_09072_b200 import _lib
import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
a, b = workloads.generate(cfg)
r = L.lcs(a, b, device=0)
lib = _lib.load()
out = (ctypes.c_uint64 * 64)()
lib.lcsg_sweep_stats.argtypes = [ctypes.c_void_p]; lib.lcsg_sweep_stats.restype = ctypes.c_int
assert lib.lcsg_sweep_stats(out) == 0
st = np.array(list(out), dtype=np.float64).reshape(8, 8)
print("lcs", r.length)
print("group threads | row steps | evaluation rounds/step | walk cells/step | splits per cell")
for c in range(8):
    s = st[c]
    if s[0] == 0:
        continue
    print(f"{32 << c:5d} | {int(s[0]):8d} | {s[1]/s[0]:.2f} | {s[2]/s[0]:.2f} | {s[3]/s[0]:.1f}")
