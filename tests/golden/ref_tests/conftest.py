"""Runs the REFERENCE's own hot-path tests against the B200 package.

The test modules next to this file (test_gram.py, test_solvers.py,
test_data.py and their helper oracles.py) are verbatim copies of
/root/reference/pkg/tests/ -- test infrastructure, vendored so the GPU box
(which has no /root/reference) can run them; they are not product code.  This
conftest replaces the reference's own (which only puts this directory on
sys.path) and, in addition, aliases the package name ``cmf`` to
``paper_1808_03843_b200`` the way INTEGRATION.md tells a user to, so the
reference's imports (``from cmf import ...``, ``from cmf.gram import ...``)
resolve to the B200 implementation.  tests/test_gpu_reference_suite.py runs
this directory under ``-m gpu``; the top-level conftest keeps plain
``pytest tests/`` from collecting it directly.
"""

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
for p in (HERE, ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import paper_1808_03843_b200 as _b200  # noqa: E402

sys.modules["cmf"] = _b200
for _sub in ("als", "data", "errors", "factors", "gram", "implicit", "parallel", "report", "solvers"):
    sys.modules["cmf." + _sub] = importlib.import_module("paper_1808_03843_b200." + _sub)
