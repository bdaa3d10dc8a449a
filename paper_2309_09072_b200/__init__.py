"""B200-native Lu-Liu grid-graph LCS (arXiv 2309.09072) -- drop-in for the
reference package ``lcsgrid``.

Same public entry points as the reference (``lcsgrid/__init__.py:10-23`` plus
the solver functions of ``solver.py``); every solve runs hand-written sm_100a
kernels through the C-ABI library ``lib/liblcsgrid_b200.so``
(``include/lcsgrid_b200.h``).  No CPU fallback, no multi-backend dispatch.

    import paper_2309_09072_b200 as lcsgrid
    lcsgrid.lcs("gatttatgcagg", "tcaggatt").length   # 5
"""

from ._backend import default_backend as active_backend
from ._backend import have_extension
from .dp import dp_lcs
from .seqcore import BreakoutRow, GridModel, LcsResult, inf_value, match_positions
from .solver import (
    CostTable,
    assemble_lcs,
    build_cost_table,
    combine_row,
    lcs,
    lcs_length,
    lcs_batch,
    reserve,
    sweep_errors,
    sweep_paths,
    trim,
    lcs_many,
    recover_cross_vertices,
)

__all__ = [
    "BreakoutRow",
    "CostTable",
    "GridModel",
    "LcsResult",
    "active_backend",
    "assemble_lcs",
    "build_cost_table",
    "combine_row",
    "dp_lcs",
    "have_extension",
    "inf_value",
    "lcs",
    "lcs_length",
    "lcs_batch",
    "reserve",
    "sweep_errors",
    "sweep_paths",
    "trim",
    "lcs_many",
    "match_positions",
    "recover_cross_vertices",
]

__version__ = "0.1.0"
