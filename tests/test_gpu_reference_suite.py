"""Drop-in conformance: the reference's OWN test suite (pkg/tests, 98 tests:
test_core.py, test_householder.py, test_trees.py) run unmodified against this
repo's drop-in package ``pkg/src/caqr`` on the GPU.

The suite is staged (not committed) into baseline/_ref/pkg_tests by
``cp -r /root/reference/pkg/tests baseline/_ref/pkg_tests`` in the build
container; baseline/_ref is git-ignored and travels to the GPU box.  The last
run's pass list is profiles/r02/reference_suite.txt.
"""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not staged in baseline/_ref")
def test_reference_suite_passes_on_the_dropin(tmp_path):
    out = tmp_path / "suite.txt"
    rc = subprocess.run([os.path.join(ROOT, "tools", "run_reference_suite.sh"), str(out)],
                        capture_output=True, text=True, timeout=1500).returncode
    text = out.read_text()
    assert rc == 0, text[-3000:]
    assert "98 passed" in text, text[-2000:]
