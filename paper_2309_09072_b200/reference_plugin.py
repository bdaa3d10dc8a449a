"""Kernel-level plugin for the UNMODIFIED reference package.

The reference selects its combine kernel through ``_backend.BACKENDS``
(reference ``_backend.py:20-22``): a name -> module map whose modules expose
``NAME`` and ``combine_level(upper_reach, upper_kmax, lower_reach,
lower_wstar, out_reach, out_trace, with_trace, inf, i_lo, i_hi)``
(reference ``_kernel.pyx:63-66``; Python twin ``_pykernel.py:51-62``).  This
module is that plugin, backed by the C-ABI ``lcsg_combine_level``
(include/lcsgrid_b200.h): a reference maintainer registers it with

    import lcsgrid._backend as B
    from paper_2309_09072_b200 import reference_plugin
    B.BACKENDS["cuda"] = reference_plugin

and every ``build_cost_table`` / ``lcs`` call with ``backend="cuda"`` (or
``LCSGRID_BACKEND=cuda``) then runs its combines on the GPU while the
reference's own Python recursion, leaf step and extraction stay in charge.
Contract kept from the reference: only rows ``[i_lo, i_hi)`` of
``out_reach`` / ``out_trace`` are written, inputs are read-only, nothing is
allocated in the caller's arrays, wrong dtypes raise ValueError.

Each call copies its tables host -> device and the row window back, so this
binding is for drop-in compatibility, not speed: the supported fast path is
the whole-solve API (``paper_2309_09072_b200.lcs`` -> ``lcsg_lcs``).
"""

from __future__ import annotations

import numpy as np

from . import _lib

NAME = "cuda"


def _c_int32(name, a, ndim):
    if not isinstance(a, np.ndarray) or a.dtype != np.intc or a.ndim != ndim:
        raise ValueError(f"{name}: expected a {ndim}-d int32 array")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous")
    return a


def combine_level(upper_reach, upper_kmax, lower_reach, lower_wstar, out_reach, out_trace,
                  with_trace, inf, i_lo, i_hi):
    """Rows [i_lo, i_hi) of one combine (reference _kernel.pyx:63-82)."""
    import torch

    U = _c_int32("upper_reach", upper_reach, 2)
    K = _c_int32("upper_kmax", upper_kmax, 1)
    Lo = _c_int32("lower_reach", lower_reach, 2)
    R = _c_int32("out_reach", out_reach, 2)
    i_lo, i_hi = int(i_lo), int(i_hi)
    if i_hi <= i_lo:
        return
    n1, w1 = R.shape
    if with_trace:
        T = _c_int32("out_trace", out_trace, 2)
        if T.shape != R.shape:
            raise ValueError("out_trace: shape differs from out_reach")
    dev = torch.device("cuda", torch.cuda.current_device())
    dU = torch.from_numpy(U).to(dev)
    dK = torch.from_numpy(K).to(dev)
    dL = torch.from_numpy(Lo).to(dev)
    dR = torch.empty((n1, w1), dtype=torch.int32, device=dev)
    dT = torch.empty((n1, w1), dtype=torch.int32, device=dev) if with_trace else None
    stream = torch.cuda.current_stream(dev)
    rc = _lib.load().lcsg_combine_level(
        dU.data_ptr(), U.shape[1], dK.data_ptr(), dL.data_ptr(), Lo.shape[1], int(lower_wstar),
        dR.data_ptr(), dT.data_ptr() if dT is not None else None, w1, int(bool(with_trace)),
        int(inf), n1, i_lo, i_hi, stream.cuda_stream)
    _lib.check(rc, "combine_level")
    R[i_lo:i_hi] = dR[i_lo:i_hi].cpu().numpy()
    if with_trace:
        out_trace[i_lo:i_hi] = dT[i_lo:i_hi].cpu().numpy()
