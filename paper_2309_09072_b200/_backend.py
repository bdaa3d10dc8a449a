"""Backend resolution (reference _backend.py:1-50), narrowed to ONE path.

The reference registers {"python", "cython"} and resolves ``backend=`` or
``LCSGRID_BACKEND``.  This package has exactly one backend -- the sm_100a
CUDA library -- and no fallback: None / "auto" / "cuda" select it.  The
reference's own names "cython" and "python" are accepted as aliases of
"cuda" (same results, bit for bit), so code written against the reference --
``backend="cython"`` or ``LCSGRID_BACKEND=python`` -- keeps working unchanged
as a drop-in; anything else raises ValueError in the reference's message
style (_backend.py:33,47-50).
"""

from __future__ import annotations

import os

from . import _lib

BACKENDS = ("cuda",)
# reference backend names (reference _backend.py:20-22) -> the one CUDA path
ALIASES = {"cython": "cuda", "python": "cuda"}


def have_extension() -> bool:
    """True when the CUDA shared library is built and loadable."""
    return _lib.available()


def default_backend() -> str:
    env = os.environ.get("LCSGRID_BACKEND")
    env = ALIASES.get(env, env)
    if env and env not in BACKENDS:
        raise ValueError(f"LCSGRID_BACKEND={env!r} not available; choices: {list(BACKENDS)}")
    return "cuda"


def resolve(name=None) -> str:
    """Map a backend name (None/'auto'/'cuda') to the CUDA path."""
    if name in (None, "auto"):
        name = default_backend()
    name = ALIASES.get(name, name)
    if name not in BACKENDS:
        raise ValueError(
            f"unknown backend {name!r}; choices: {sorted(BACKENDS + tuple(ALIASES))} "
            "(the CUDA kernel is only available after building the extension)")
    return name
