"""Build the library of an older commit as an A/B variant:
    python tools/ab_commit.py COMMIT NAME  -> paper_2309_09072_b200/lib/ab/NAME.so"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_09072_b200 import _lib  # noqa: E402

commit, name = sys.argv[1], sys.argv[2]
with tempfile.TemporaryDirectory() as tmp:
    subprocess.run(f"git -C {ROOT} archive {commit} paper_2309_09072_b200/csrc include | tar -x -C {tmp}",
                   shell=True, check=True)
    _lib.CSRC = os.path.join(tmp, "paper_2309_09072_b200", "csrc")
    srcs = [s for s in _lib.SOURCES if os.path.exists(os.path.join(_lib.CSRC, s))]
    _lib.SOURCES = srcs
    print(_lib.build_library(out=os.path.join(_lib.LIB_DIR, "ab", name + ".so")))
