"""Build experiment variants of the library with extra -D defines, for A/B
timing on the GPU box (LCSG_LIB_PATH selects one per process):

    python tools/ab_build.py NAME=DEF1,DEF2 NAME2= ...
    -> paper_2309_09072_b200/lib/ab/NAME.so
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_09072_b200 import _lib  # noqa: E402

jobs = []
for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    out = os.path.join(_lib.LIB_DIR, "ab", name + ".so")
    jobs.append((out, [d for d in defs.split(",") if d]))
with ThreadPoolExecutor(max_workers=2) as ex:
    for path in ex.map(lambda j: _lib.build_library(out=j[0], defines=j[1]), jobs):
        print("built", path)
