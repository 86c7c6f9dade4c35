"""The reference's own hot-path tests (test_gram.py, test_solvers.py,
test_data.py from /root/reference/pkg/tests, vendored verbatim under
tests/golden/ref_tests) run UNCHANGED against this package on the B200,
through the ``cmf`` import alias of INTEGRATION.md.  VERDICT r1 "next" #3:
the reference's ~45 hot-path tests must pass on the GPU."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SUITE = os.path.join(HERE, "golden", "ref_tests")


@pytest.mark.parametrize("module", ["test_gram.py", "test_solvers.py", "test_data.py"])
def test_reference_suite_passes(cuda_device, module):
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        "--rootdir", SUITE, os.path.join(SUITE, module)],
                       cwd=SUITE, capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
