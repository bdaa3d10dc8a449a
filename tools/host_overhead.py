"""Host-side cost of one lcsg_build call (enqueue only) vs the device time."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_09072_b200 import _lib
import workloads
lib = _lib.load()
a, b = workloads.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
r = np.frombuffer(a, np.uint8); c = np.frombuffer(b, np.uint8)
s = torch.cuda.current_stream()
for it in range(4):
    h = ctypes.c_void_p()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    rc = lib.lcsg_build(r.ctypes.data, len(a), c.ctypes.data, len(b), 1, len(a) + 1, 1 | 2, 0,
                        ctypes.c_void_p(s.cuda_stream), ctypes.byref(h))
    t1 = time.perf_counter()
    length = ctypes.c_int32(); k = min(len(a), len(b))
    sub = np.empty(k, np.uint8); rp = np.empty(k, np.int32); cp = np.empty(k, np.int32)
    lib.lcsg_extract(h, -1, ctypes.byref(length), sub.ctypes.data, rp.ctypes.data, cp.ctypes.data)
    e1.record(s); torch.cuda.synchronize()
    st = [ctypes.c_int64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64()]
    lib.lcsg_stats(h, *[ctypes.byref(x) for x in st])
    print(f"build enqueue {1e3*(t1-t0):.2f} ms host; step {e0.elapsed_time(e1):.2f} ms device; "
          f"leaf {st[2].value:.2f} combine {st[1].value:.2f} total(build+extract) {st[3].value:.2f}")
    lib.lcsg_free(h)
