"""Backend resolution (reference _backend.py:1-50), narrowed to ONE path.

The reference registers {"python", "cython"} and resolves ``backend=`` or
``LCSGRID_BACKEND``.  This package has exactly one backend -- the sm_100a
CUDA library -- and no fallback: None / "auto" / "cuda" select it, anything
else raises ValueError in the reference's message style (_backend.py:47-50).
"""

from __future__ import annotations

import os

from . import _lib

BACKENDS = ("cuda",)


def have_extension() -> bool:
    """True when the CUDA shared library is built and loadable."""
    return _lib.available()


def default_backend() -> str:
    env = os.environ.get("LCSGRID_BACKEND")
    if env and env not in BACKENDS:
        raise ValueError(f"LCSGRID_BACKEND={env!r} not available; choices: {list(BACKENDS)}")
    return "cuda"


def resolve(name=None) -> str:
    """Map a backend name (None/'auto'/'cuda') to the CUDA path."""
    if name in (None, "auto"):
        name = default_backend()
    if name not in BACKENDS:
        raise ValueError(
            f"unknown backend {name!r}; choices: {list(BACKENDS)} "
            "(the CUDA kernel is only available after building the extension)")
    return name
