import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libwadg_b200.so")


@pytest.fixture
def rng():
    # the reference tests' seed (R/pkg/tests/conftest.py:40-42)
    return np.random.default_rng(1234)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def het_c2(*xyz):
    return 1.0 + 0.5 * np.sin(np.pi * np.hypot(xyz[0], xyz[1]))


def golden_mesh(g):
    from paper_1608_03836_b200 import meshgen, refelem
    shape = refelem.ElementShape(str(g["shape"]))
    return meshgen.CurvedMesh(shape, int(g["N_geo"]), g["elem_map_nodes"], g["face_connectivity"],
                              g["boundary_tags"], h=float(g["h"]))


GOLDEN_CASES = {
    # name: (c2, heterogeneous?)
    "config1_tri": 1.0,
    "tri_strong_het": het_c2,
    "quad_sw": 1.0,
    "quad_strong": het_c2,
    "tri_exact": het_c2,          # ExactCurvedMass comparator
}
