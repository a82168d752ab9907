"""pytest plugin: run the reference's own solver tests
(R/pkg/tests/test_solver.py) against this package.

Installs a ``wadg.solver`` module whose API is ``paper_1608_03836_b200.solver``
(the drop-in; every RHS / stage / run goes through libwadg_b200.so), next to
the reference's own ``wadg.meshgen`` / ``refelem`` / ``geometry`` /
``operators`` (the tests build their meshes and reference elements with
them).  The only adapters are at the type boundary: reference mesh objects
and ElementShape enum members are converted by value, and ``stable_dt``
rebuilds the reference element in this package.  Used by
tests/test_reference_suite.py; the reference package comes from
baseline/_ref (the offline install, git-ignored), its tests from a copy
placed there by tests/refsuite/stage_reference_tests.py.
"""

import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

import wadg  # noqa: E402  (the reference package)
import wadg.meshgen  # noqa: E402,F401
import wadg.refelem  # noqa: E402,F401
from paper_1608_03836_b200 import meshgen as _M  # noqa: E402
from paper_1608_03836_b200 import refelem as _R  # noqa: E402
from paper_1608_03836_b200 import solver as _S  # noqa: E402


def _shape(s):
    return _R.ElementShape(s.value)


def _mesh(m):
    if isinstance(m, _M.CurvedMesh):
        return m
    return _M.CurvedMesh(_shape(m.shape), m.N_geo, m.elem_map_nodes, m.face_connectivity, m.boundary_tags,
                         h=m.h, provenance=dict(getattr(m, "provenance", {}) or {}))


def _build():
    sv = types.ModuleType("wadg.solver")
    sv.__doc__ = "paper_1608_03836_b200.solver behind the reference's wadg.solver name (test shim)"
    for name in dir(_S):
        if not name.startswith("__"):
            setattr(sv, name, getattr(_S, name))

    class Discretization(_S.Discretization):
        def __init__(self, mesh, config, medium=_S.MediumField(), **kw):
            super().__init__(_mesh(mesh), config, medium, **kw)

    def sufficient_quadrature_degrees(N, N_geo, shape):
        return _S.sufficient_quadrature_degrees(N, N_geo, _shape(shape))

    def stable_dt(mesh, ref, medium, cfl):
        ours = _R.build_reference_element(ref.N, _shape(ref.shape))
        return _S.stable_dt(_mesh(mesh), ours, medium, cfl)

    def run(mesh, config, initial_fn, T, *a, **kw):
        return _S.run(_mesh(mesh), config, initial_fn, T, *a, **kw)

    def project_initial_condition(mesh, config, initial_fn, *a, **kw):
        return _S.project_initial_condition(_mesh(mesh), config, initial_fn, *a, **kw)

    sv.Discretization = Discretization
    sv.sufficient_quadrature_degrees = sufficient_quadrature_degrees
    sv.stable_dt = stable_dt
    sv.run = run
    sv.project_initial_condition = project_initial_condition
    return sv


sys.modules["wadg.solver"] = wadg.solver = _build()


def pytest_report_header(config):
    return "wadg.solver -> paper_1608_03836_b200.solver (reference tests against the drop-in)"
