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


# measured parity errors, printed in the terminal summary (also under -q) and
# written to gpurun_out/parity_errors.jsonl when that directory exists
_PARITY = []


def record_parity(case, err, tol):
    _PARITY.append({"case": case, "rel_l2": float(err), "tol": float(tol)})


def pytest_terminal_summary(terminalreporter):
    if not _PARITY:
        return
    terminalreporter.write_sep("-", "measured parity (relative L2 vs the fp64 oracle)")
    for r in _PARITY:
        terminalreporter.write_line(f"{r['rel_l2']:.3e}  (bar {r['tol']:.0e})  {r['case']}")
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        import json
        with open(os.path.join(out, "parity_errors.jsonl"), "a") as f:
            for r in _PARITY:
                f.write(json.dumps(r) + "\n")


def submesh(mesh, elems):
    """The sample elements and their face neighbours as a standalone mesh.
    Faces leading out of the patch become boundary faces; that only changes
    the right-hand side of the neighbours, never of the sample elements."""
    from paper_1608_03836_b200 import meshgen
    conn = mesh.face_connectivity
    nb = conn[elems, :, 0]
    patch = np.unique(np.concatenate([elems, nb[nb >= 0]]))
    index = np.full(mesh.K, -1, dtype=np.int64)
    index[patch] = np.arange(len(patch))
    c = conn[patch].copy()
    inside = c[:, :, 0] >= 0
    inside[inside] = index[c[:, :, 0][inside]] >= 0
    c[:, :, 0] = np.where(inside, index[np.maximum(c[:, :, 0], 0)], -1)
    c[:, :, 1] = np.where(inside, c[:, :, 1], -1)
    tags = np.where(inside, 0, np.maximum(mesh.boundary_tags[patch], 1))
    ori = np.where(inside, mesh.face_orientation[patch], 0)
    sub = meshgen.CurvedMesh(mesh.shape, mesh.N_geo, mesh.elem_map_nodes[patch], c, tags, h=mesh.h,
                             face_orientation=ori)
    return sub, patch, index[elems]


@pytest.fixture(autouse=True)
def _release_device_memory():
    """GPU tests build full-size (1.5M-tet) problems one after another: collect
    the previous test's objects (a HostPipeline / HaloExchange refers back to its
    Discretization) and return the cached blocks before the next test."""
    yield
    import gc
    gc.collect()
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.empty_cache()
    except Exception:
        pass
