"""Copy the reference's solver tests (R/pkg/tests/test_solver.py and its
conftest) into baseline/_ref/tests/, next to the reference install, so that
they travel to the GPU box (baseline/_ref is git-ignored: the reference's
files never enter this repository's history).  Run in the build container,
where /root/reference exists."""

import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref", "tests")


def stage():
    if not os.path.isdir(SRC):
        return False
    os.makedirs(DST, exist_ok=True)
    for f in ("test_solver.py", "conftest.py"):
        shutil.copyfile(os.path.join(SRC, f), os.path.join(DST, f))
    return True


if __name__ == "__main__":
    print("staged" if stage() else "no reference tree")
