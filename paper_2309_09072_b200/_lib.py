"""Loader and ctypes bindings of the C-ABI library (include/lcsgrid_b200.h).

The library is built in-tree (``paper_2309_09072_b200/lib/liblcsgrid_b200.so``)
by :func:`build_library` / ``__graft_entry__.build()``.  There is no CPU
fallback: if the shared object is missing or no GPU is visible every solve
raises, loudly.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
LIB_DIR = os.path.join(_PKG, "lib")
_DEFAULT_LIB = os.path.join(LIB_DIR, "liblcsgrid_b200.so")
LIB_PATH = os.environ.get("LCSG_LIB_PATH") or _DEFAULT_LIB
CSRC = os.path.join(_PKG, "csrc")
SOURCES = ["lcsg_api.cu", "lcsg_kernels.cu", "lcsg_refine.cu", "lcsg_tile.cu", "lcsg_narrow.cu",
           "lcsg_probe.cu", "lcsg_sweep.cu"]
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
]

LCSG_OK = 0
LCSG_EINVAL = -1
LCSG_ECUDA = -2
LCSG_ENOMEM = -3
LCSG_ENODEV = -4
LCSG_ERANGE = -5
LCSG_WITH_TRACE = 1
LCSG_TIMING = 2

_lib = None
_lock = threading.Lock()

_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32

# name -> (restype, argtypes); every symbol declared in include/lcsgrid_b200.h
SIGNATURES = {
    "lcsg_last_error": (ctypes.c_char_p, []),
    "lcsg_abi_version": (ctypes.c_int, []),
    "lcsg_device_count": (ctypes.c_int, []),
    "lcsg_build": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i32, _i32, ctypes.c_uint32, ctypes.c_int,
                                  _vp, ctypes.POINTER(_vp)]),
    "lcsg_build_device": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i32, _i32, ctypes.c_uint32,
                                         ctypes.c_int, _vp, ctypes.POINTER(_vp)]),
    "lcsg_free": (ctypes.c_int, [_vp]),
    "lcsg_trim": (ctypes.c_int, [ctypes.c_int]),
    "lcsg_reserve": (ctypes.c_int, [ctypes.c_int, _i64]),
    "lcsg_sync": (ctypes.c_int, [_vp]),
    "lcsg_num_nodes": (_i32, [_vp]),
    "lcsg_root": (_i32, [_vp]),
    "lcsg_node_info": (ctypes.c_int, [_vp, _i32, _i32p]),
    "lcsg_node_wstar": (ctypes.c_int, [_vp, _i32, _i32p]),
    "lcsg_node_reach": (ctypes.c_int, [_vp, _i32, _vp]),
    "lcsg_node_trace": (ctypes.c_int, [_vp, _i32, _vp]),
    "lcsg_node_kmax": (ctypes.c_int, [_vp, _i32, _vp]),
    "lcsg_node_reach_device": (ctypes.c_int, [_vp, _i32, ctypes.POINTER(_vp)]),
    "lcsg_length": (ctypes.c_int, [_vp, _i32p]),
    "lcsg_recover": (ctypes.c_int, [_vp, _i32, _vp]),
    "lcsg_extract": (ctypes.c_int, [_vp, _i32, _i32p, _vp, _vp, _vp]),
    "lcsg_assemble": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, ctypes.c_int, _i32p, _vp, _vp,
                                     _vp]),
    "lcsg_lcs": (ctypes.c_int, [_vp, _i64, _vp, _i64, ctypes.c_uint32, ctypes.c_int, _vp, _i32p,
                                _vp, _vp, _vp]),
    "lcsg_lcs_device": (ctypes.c_int, [_vp, _i64, _vp, _i64, ctypes.c_uint32, ctypes.c_int, _vp,
                                       _i32p, _vp, _vp, _vp]),
    "lcsg_lcs_batch": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i32, ctypes.c_uint32, ctypes.c_int,
                                      _vp, _vp, _vp, _vp, _vp]),
    "lcsg_lcs_batch_device": (ctypes.c_int, [_vp, _i64, _vp, _i64, _i32, ctypes.c_uint32,
                                             ctypes.c_int, _vp, _vp, _vp, _vp, _vp]),
    "lcsg_combine_level": (ctypes.c_int, [_vp, _i32, _vp, _vp, _i32, _i32, _vp, _vp, _i32,
                                          ctypes.c_int, _i32, _i64, _i64, _i64, _vp]),
    "lcsg_base_case_row": (ctypes.c_int, [_vp, _i64, ctypes.c_uint8, _vp, _vp]),
    "lcsg_combine_rows": (ctypes.c_int, [_vp, _i32, _vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp,
                                         _vp, _i32, _i32, _i64, _i64, _i64, _vp]),
    "lcsg_recover_from": (ctypes.c_int, [_vp, _i32, _i32, _vp]),
    "lcsg_sweep_errors": (ctypes.c_int, [ctypes.c_int, _i32p, ctypes.c_int]),
    "lcsg_sweep_paths": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                        ctypes.c_int]),
    "lcsg_probe_int32_rate": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                             _i32p, ctypes.POINTER(ctypes.c_double)]),
    "lcsg_stats": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
                                  ctypes.POINTER(_i64)]),
}


def build_library(verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the CUDA sources for sm_100a into the in-tree shared object
    (one nvcc per translation unit in parallel, then one link).  ``out`` /
    ``defines`` build an experiment variant elsewhere (tools/ab_build.py)."""
    from concurrent.futures import ThreadPoolExecutor

    out = out or LIB_PATH
    os.makedirs(os.path.dirname(out), exist_ok=True)
    obj_dir = os.path.join(os.path.dirname(out), "obj" if out == LIB_PATH else
                           "obj_" + os.path.basename(out)[:-3])
    os.makedirs(obj_dir, exist_ok=True)
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"] + [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        cmd = ["nvcc", *compile_flags, "-c", "-o", obj, src]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        results = list(ex.map(compile_one, srcs))
    log = ""
    for obj, res in results:
        log += res.stdout + res.stderr
        if res.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    cmd = ["nvcc", *NVCC_FLAGS, "-o", out, *[o for o, _ in results]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(log + res.stdout + res.stderr)
    return out


def load():
    """Load the shared object (once).  Raises if it is absent: no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                    "(the CUDA path has no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                if LIB_PATH != _DEFAULT_LIB and not hasattr(lib, name):
                    continue  # an older A/B build (tools/ab_commit.py)
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def available() -> bool:
    try:
        load()
        return True
    except OSError:
        return False
    except ImportError:
        return False


def last_error() -> str:
    return load().lcsg_last_error().decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == LCSG_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == LCSG_ERANGE or rc == LCSG_EINVAL:
        raise ValueError(msg)
    if rc == LCSG_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)
