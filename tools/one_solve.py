"""One (or a few) cfg solves through the C-ABI (build + extract), for ncu
launch lists: `ncu --metrics gpu__time_duration.sum --csv python tools/one_solve.py 5`."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2309_09072_b200 import _lib
import workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1
lib = _lib.load()
a, b = workloads.generate(cfg)
r = np.frombuffer(a, np.uint8); c = np.frombuffer(b, np.uint8)
s = torch.cuda.current_stream()
for _ in range(iters):
    h = ctypes.c_void_p()
    _lib.check(lib.lcsg_build(r.ctypes.data, len(a), c.ctypes.data, len(b), 1, len(a) + 1, 1, 0,
                                   ctypes.c_void_p(s.cuda_stream), ctypes.byref(h)))
    length = ctypes.c_int32(); k = min(len(a), len(b))
    sub = np.empty(k, np.uint8); rp = np.empty(k, np.int32); cp = np.empty(k, np.int32)
    _lib.check(lib.lcsg_extract(h, -1, ctypes.byref(length), sub.ctypes.data, rp.ctypes.data,
                                     cp.ctypes.data))
    lib.lcsg_free(h)
print("length", length.value)
