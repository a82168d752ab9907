"""The reference's own solver tests (R/pkg/tests/test_solver.py, 24 tests)
run against the drop-in through tests/refsuite/wadg_shim.py: the reference's
``wadg.solver`` name resolves to paper_1608_03836_b200.solver, whose compute
goes through libwadg_b200.so.  Needs the GPU and the reference install with
its staged tests under baseline/_ref (tests/refsuite/stage_reference_tests.py)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests", "test_solver.py")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(REF_TESTS), reason="reference tests not staged under baseline/_ref")
def test_reference_solver_suite_passes_against_drop_in():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         os.path.join(ROOT, "baseline", "_ref"), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    out = subprocess.run([sys.executable, "-m", "pytest", REF_TESTS, "-p", "wadg_shim", "-q",
                          "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir",
                          os.path.dirname(REF_TESTS)],
                         cwd=os.path.dirname(REF_TESTS), env=env, capture_output=True, text=True, timeout=1800)
    print(out.stdout[-3000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "24 passed" in out.stdout
