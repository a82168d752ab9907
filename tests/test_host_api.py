"""Host-side behaviour of the drop-in API (no GPU needed): configuration
errors and types match the reference (R/pkg/src/wadg/solver.py), and the
device path refuses to run without CUDA (there is no CPU fallback)."""

import numpy as np
import pytest
import torch

from paper_1608_03836_b200 import meshgen, refelem, solver
from paper_1608_03836_b200.refelem import ElementShape
from paper_1608_03836_b200.solver import (ConfigError, FieldState, FluxParams, Formulation, MassMode,
                                          MediumField, SolverConfig)


def test_flux_params_validation():
    with pytest.raises(ConfigError):
        FluxParams(-0.1, 0.0)
    assert issubclass(ConfigError, ValueError)


def test_nonpositive_wavespeed_rejected():
    with pytest.raises(ConfigError):
        solver.Discretization(meshgen.uniform_quad_mesh(2), SolverConfig(N=2), MediumField(-1.0))
    # a callable medium is checked where it is evaluated (on the device's points),
    # with the reference's ConfigError (R/pkg/src/wadg/solver.py:62-63)
    from paper_1608_03836_b200.device import medium_on_device
    x = torch.linspace(-1, 1, 7, dtype=torch.float64)
    with pytest.raises(ConfigError):
        medium_on_device(lambda x, y: x, (x, x), x.shape)
    with pytest.raises(ConfigError):
        medium_on_device(lambda x, y: np.cos(x) * np.nan, (x, x), x.shape)
    v = medium_on_device(lambda x, y: 1.0 + x * x, (x, x), x.shape)        # torch expression
    w = medium_on_device(lambda x, y: 1.0 + np.asarray(x) ** 2, (x, x), x.shape)
    assert torch.equal(v, w)


def test_insufficient_quadrature_rejected():
    mesh = meshgen.uniform_quad_mesh(2, N_geo=3)     # quads need 2N + N_geo - 1 = 8
    with pytest.raises(ConfigError):
        solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.Strong, volume_quad_degree=7))
    solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.Strong, volume_quad_degree=7,
                                             face_quad_degree=7, unsafe_quadrature=True))


def test_bad_dtype_and_exact_mass_mode():
    mesh = meshgen.warped_triangle_mesh(2, 2)
    with pytest.raises(ConfigError):
        solver.Discretization(mesh, SolverConfig(N=2, dtype="float16"))
    # the ExactCurvedMass comparator is accepted; WADG mode stores no dense matrices
    # (R/pkg/tests/test_solver.py:128-133)
    dE = solver.Discretization(mesh, SolverConfig(N=2, mass_mode=MassMode.ExactCurvedMass))
    assert dE.exact_mass
    dW = solver.Discretization(mesh, SolverConfig(N=2))
    assert dW.mass_inv_p is None and dW.mass_inv_u is None


def test_sufficient_quadrature_degrees():
    assert solver.sufficient_quadrature_degrees(3, 3, ElementShape.Triangle) == (7, 8)
    assert solver.sufficient_quadrature_degrees(3, 3, ElementShape.Quadrilateral) == (8, 8)
    # paper's 4N-3 / 4N-2 at N_geo = N for tetrahedra
    assert solver.sufficient_quadrature_degrees(4, 4, ElementShape.Tetrahedron) == (13, 14)


def test_fieldstate_reference_positional_time():
    st = FieldState(np.zeros((1, 1)), np.zeros((1, 1)), np.zeros((1, 1)), 0.5)
    assert st.t == 0.5 and st.u3 is None and len(st.fields()) == 3
    st3 = FieldState.from_fields([np.zeros((1, 1))] * 4, 1.0)
    assert len(st3.fields()) == 4 and st3.t == 1.0
    with pytest.raises(FloatingPointError):
        FieldState(np.array([[np.nan]]), np.zeros((1, 1)), np.zeros((1, 1))).check_finite()


def test_discretization_host_attributes():
    mesh = meshgen.warped_cube_tet_mesh(2, 3)
    disc = solver.Discretization(mesh, SolverConfig(N=3, formulation=Formulation.StrongWeak))
    assert disc.mass_inv_p is None and disc.mass_inv_u is None
    assert disc.w_upd_p.shape == (mesh.K, disc.ref_upd.Nq)
    assert disc.bc_mask.shape == (mesh.K, 4 * disc.ref.nfq)
    # WADG storage: 2 Nq_u words per element vs 2 Np^2 for dense M_J^-1
    assert disc.ref.Np ** 2 / disc.ref_upd.Nq == pytest.approx(400 / 64)


def test_stable_dt_matches_reference_formula():
    """R/pkg/tests/test_solver.py:221-227: N=1 uniform quads, h=0.5."""
    m = meshgen.uniform_quad_mesh(4, domain=((0, 2), (0, 2)))
    ref = refelem.build_reference_element(1, ElementShape.Quadrilateral)
    assert solver.stable_dt(m, ref, MediumField(1.0), cfl=1.0) == pytest.approx(0.25 / 4, rel=1e-12)
    with pytest.raises(ConfigError):
        solver.stable_dt(m, ref, MediumField(1.0), cfl=0.0)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_cuda():
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    disc = solver.Discretization(mesh, SolverConfig(N=2, formulation=Formulation.StrongWeak))
    st = FieldState.from_fields([np.zeros((mesh.K, disc.ref.Np))] * 4)
    with pytest.raises(RuntimeError, match="CUDA"):
        solver.rhs_full(st, disc)
    with pytest.raises(RuntimeError, match="CUDA"):
        solver.lsrk_step(st, 1e-3, disc.rhs)
    with pytest.raises(RuntimeError, match="CUDA"):
        solver.project_initial_condition(mesh, disc.config, lambda x, y, z: (0 * x,) * 4)
