"""Face matching pinned by physical continuity, independent of the shared
setup's permutation tables.

On a conforming curved tetrahedral mesh with N_geo = N the solution nodes are
the map nodes, so the nodal interpolant of any smooth function f (values
f(x_node)) is continuous across every interior face: both sides' face nodes sit
at the same physical points and carry the same values, and each side's trace
is the degree-N interpolant of those values on the face.  In the strong form
every interior-face flux is a jump ([u.n] - tau_p [p], [p] - tau_u [u.n],
R/pkg/src/wadg/solver.py:220-232), so the surface term of an element with no
boundary face vanishes for such a state.  A wrong face-orientation permutation
(ext_node / fperm / face_orientation), a wrong neighbour face, or a wrong trace
gather makes it O(1).  The mesh has several orientation codes; the check covers
every one of them, the oracle's exterior evaluation (CPU) and the GPU's
per-phase surface kernel and fused stages (the reference 2D tests the same
property through its constant-state test, R/pkg/tests/test_solver.py:33-48,
which a permutation cannot fail)."""

import numpy as np
import pytest

import wadg_oracle as O
from paper_1608_03836_b200 import meshgen
from paper_1608_03836_b200.solver import FieldState, FluxParams, Formulation, SolverConfig


def _smooth_state(mesh):
    x, y, z = (mesh.elem_map_nodes[..., i] for i in range(3))
    p = np.sin(1.3 * x + 0.4) * np.cos(0.7 * y) + z ** 3
    u = [np.cos(x * y) + 0.3 * z, x ** 2 - y * z, np.sin(2.0 * z) + 0.5 * x]
    return p, u


def _interior(mesh):
    return ~(mesh.face_connectivity[:, :, 0] < 0).any(axis=1)


def _orientation_codes(mesh):
    inner = mesh.face_connectivity[:, :, 0] >= 0
    return set(map(tuple, np.stack([mesh.face_connectivity[..., 1][inner],
                                    mesh.face_orientation[inner]], axis=1).tolist()))


@pytest.mark.parametrize("N", [2, 3])
def test_oracle_interior_surface_term_vanishes_for_continuous_fields(N):
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    assert mesh.N_geo == N
    assert len(_orientation_codes(mesh)) > 1
    od = O.OracleDiscretization(mesh, N, False, tau_p=1.0, tau_u=1.0)
    p, u = _smooth_state(mesh)
    rp, ru = O.surface_terms(O.State(p, u), od)
    inner = _interior(mesh)
    assert inner.sum() > 0
    scale = max(np.abs(rp).max(), max(np.abs(a).max() for a in ru))
    assert scale > 1e-2                                    # boundary faces do contribute
    for a in [rp] + list(ru):
        assert np.abs(a[inner]).max() < 1e-10 * scale
    # a discontinuous state (the same fields, one element perturbed) is seen
    p2 = p.copy()
    p2[np.nonzero(inner)[0][0]] += 1.0
    rp2, _ = O.surface_terms(O.State(p2, u), od)
    assert np.abs(rp2[inner]).max() > 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 2e-5)])
@pytest.mark.parametrize("N", [2, 3, 4])
def test_gpu_interior_surface_term_vanishes_for_continuous_fields(N, dtype, tol):
    """The per-phase surface kernel (strong form), and the fused stage of the
    default kernel (strong form where it exists, N = 2..4) through
    rhs_full - M^-1 volume: interior elements see no flux for a continuous state."""
    from paper_1608_03836_b200 import solver
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.Strong, flux=FluxParams(1.0, 1.0), dtype=dtype)
    disc = solver.Discretization(mesh, cfg)
    p, u = _smooth_state(mesh)
    st = FieldState(p, *u)
    inner = _interior(mesh)
    surf = solver._surface_terms(st, disc, False)
    scale = max(np.abs(np.asarray(a)).max() for a in surf)
    assert scale > 1e-2
    for a in surf:
        assert np.abs(np.asarray(a)[inner]).max() < tol * scale
    # the fused stage gathers exterior traces itself: rhs_full = M^-1 (volume + surface)
    assert disc.dev.fused is not None
    full = solver.rhs_full(st, disc).fields()
    vol = solver._volume_terms(st, disc, False)
    mv = solver.apply_mass_inverse(FieldState(*vol), disc).fields()
    big = max(np.abs(np.asarray(a)).max() for a in full)
    for a, b in zip(full, mv):
        assert np.abs((np.asarray(a) - np.asarray(b))[inner]).max() < 10 * tol * big


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 2e-5)])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_gpu_fused_strong_weak_interior_flux_is_continuous_part_only(N, dtype, tol):
    """Strong-weak form (the fused kernels of the headline path: register
    stage, tcgen05, DMMA, mma.sync): for a continuous state the interior-face
    flux reduces to its average part {u.n}, which both sides see with opposite
    normals.  Checked against the oracle's strong-weak rhs on the same state,
    so a face-matching error in any fused kernel shows as an O(1) difference."""
    from paper_1608_03836_b200 import solver
    mesh = meshgen.warped_cube_tet_mesh(3, N)
    cfg = SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(1.0, 1.0), dtype=dtype)
    disc = solver.Discretization(mesh, cfg)
    assert disc.dev.fused is not None
    p, u = _smooth_state(mesh)
    got = [np.asarray(a) for a in solver.rhs_full(FieldState(p, *u), disc).fields()]
    od = O.OracleDiscretization(mesh, N, True, tau_p=1.0, tau_u=1.0)
    want = O.rhs_full(O.State(p, u), od).fields()
    big = max(np.abs(a).max() for a in want)
    for a, b in zip(got, want):
        assert np.abs(a - b).max() < 10 * tol * big
