"""Shared test setup: markers, import paths, golden fixtures.

`-m "not gpu"` tests run on the CPU build container (oracle vs goldens, host
logic, C-ABI exports); `-m gpu` tests are the parity tests proper and call
the CUDA path through the C-ABI on a B200.  The oracle (oracle/) is imported
here as the CHECKER only.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle"), GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: full-size configs (minutes)")


def load_npz_trees(path):
    """{prefix: [node dicts in reference post-order]} from a make_golden dump."""
    z = np.load(path)
    out = {}
    for key in z.files:
        if key.endswith("/count"):
            prefix = key[: -len("/count")]
            nodes = []
            for idx in range(int(z[key])):
                base = f"{prefix}/{idx}"
                top, bottom, wstar = (int(v) for v in z[base + "/rows"])
                nodes.append({"top": top, "bottom": bottom, "wstar": wstar,
                              "reach": z[base + "/reach"], "kmax": z[base + "/kmax"],
                              "trace": z[base + "/trace"] if base + "/trace" in z.files else None})
            out[prefix] = nodes
    meta = json.loads(bytes(z["meta"]).decode()) if "meta" in z.files else None
    extra = {k: z[k] for k in z.files if k.endswith("/lcs")}
    return out, meta, extra


@pytest.fixture(scope="session")
def ref_trees():
    return load_npz_trees(os.path.join(GOLDEN, "ref_trees.npz"))


@pytest.fixture(scope="session")
def paper_tree():
    return load_npz_trees(os.path.join(GOLDEN, "paper_grid.npz"))


@pytest.fixture(scope="session")
def ref_lcs_pairs():
    with open(os.path.join(GOLDEN, "ref_lcs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def spec_examples():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def config_digests():
    with open(os.path.join(GOLDEN, "config_digests.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def reference():
    """The real reference (oracle/_ref/lcsgrid_ref, built from /root/reference
    by oracle/build_ref.sh), or skip when it was not built."""
    if not os.path.isdir(os.path.join(REF_DIR, "lcsgrid_ref")):
        pytest.skip("oracle/_ref not built (run oracle/build_ref.sh where /root/reference exists)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import lcsgrid_ref

    return lcsgrid_ref


@pytest.fixture(autouse=True)
def _sweep_invariants(request):
    """After every GPU test: the row-sweep kernels' invariant counter is zero."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    import paper_2309_09072_b200 as L

    if not L.have_extension():
        return
    try:
        import torch

        if not torch.cuda.is_available():
            return
    except Exception:
        return
    assert L.sweep_errors(reset=True) == 0, "row-sweep invariant violated"
