"""The reference-side ctypes binding shown in INTEGRATION.md §2 runs as
written: its code block is extracted from the document and its rhs_full is
checked against solver.rhs_full (which goes through the same ABI)."""

import os
import re

import numpy as np
import pytest

from paper_1608_03836_b200 import meshgen, solver
from paper_1608_03836_b200.solver import FieldState, FluxParams, Formulation, SolverConfig

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sample_module():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# wadg/_b200\.py.*?)```", text, re.S).group(1)
    ns = {}
    exec(compile(code, "INTEGRATION.md:wadg/_b200.py", "exec"), ns)
    return ns


def test_integration_binding_sample_runs(rng):
    ns = _sample_module()
    mesh = meshgen.warped_triangle_mesh(4, 3)
    cfg = SolverConfig(N=3, formulation=Formulation.StrongWeak, flux=FluxParams(0.8, 1.2))
    disc = ns["make_gpu_discretization"](mesh, cfg, solver.MediumField(1.0))
    st = FieldState(*(rng.standard_normal((mesh.K, disc.ref.Np)) for _ in range(3)))
    got = ns["rhs_full"](st, disc)
    want = solver.rhs_full(st, disc)
    for a, b in zip(got.fields(), want.fields()):
        assert np.max(np.abs(np.asarray(a) - np.asarray(b))) == 0.0
