"""Run the reference's own test files, unmodified, against this package.

The files next to this one are verbatim copies of the reference's tests
(pkg/tests/helpers.py, test_fusion.py, test_rasterizer.py,
test_renderback.py, test_acceptance.py and pkg/bindings/tests/test_session.py;
see README.md).  They import ``texelfuse`` and ``texelfuse_bindings``; here
those names are aliases of ``paper_2111_11103_b200`` and its session module,
so every fusion, rasterization and render call they make runs the sm_100a
kernels.  All of them need the GPU (marked ``gpu``).
"""

import importlib
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)  # `from helpers import ...`

import paper_2111_11103_b200 as _pkg  # noqa: E402

sys.modules["texelfuse"] = _pkg
for _name in ("cli", "errors", "formats", "fusion", "geometry", "meshio", "rasterizer", "renderback", "synthgen"):
    sys.modules["texelfuse." + _name] = importlib.import_module("paper_2111_11103_b200." + _name)
sys.modules["texelfuse_bindings"] = importlib.import_module("paper_2111_11103_b200.session")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)
