"""Evolution-operator spectra (R/pkg/src/wadg/analysis.py:22-123).

CPU: the eigen-solve and result container, restating R/pkg/tests/test_analysis.py
(TestEigenspectrum).  GPU: the device-assembled evolution matrix against the
oracle's column-by-column assembly, linearity, and the reference's spectral
invariants (skew for central flux, dissipative for upwind/penalty flux) in 2D
and on tetrahedra (R/pkg/tests/test_analysis.py TestEvolutionMatrix)."""

import csv

import numpy as np
import pytest

import wadg_oracle as O
from paper_1608_03836_b200 import analysis as an
from paper_1608_03836_b200 import meshgen
from paper_1608_03836_b200.solver import FieldState, FluxParams, Formulation, SolverConfig


def test_zero_matrix():
    spec = an.eigenspectrum(np.zeros((12, 12)))
    assert np.max(np.abs(spec.eigenvalues)) == 0.0


def test_failure_on_nonfinite():
    with pytest.raises(an.EigenSolveFailure):
        an.eigenspectrum(np.full((4, 4), np.nan))


def test_sorted_by_magnitude():
    spec = an.eigenspectrum(np.diag([1.0, -3.0, 2.0]))
    assert np.abs(spec.eigenvalues[0]) == pytest.approx(3.0)
    assert spec.max_real_part == pytest.approx(2.0)
    assert spec.spectral_radius == pytest.approx(3.0)


def test_csv(tmp_path):
    spec = an.eigenspectrum(np.diag([1.0, -2.0]))
    path = tmp_path / "s.csv"
    spec.to_csv(path)
    rows = list(csv.reader(open(path)))
    assert rows[0] == ["re", "im"]
    assert len(rows) == 3


def oracle_matrix(mesh, N, sw, tau):
    od = O.OracleDiscretization(mesh, N, sw, tau, tau)
    K, Np, fld = mesh.K, od.ref.Np, mesh.shape.dim + 1
    n = fld * K * Np
    A = np.empty((n, n))
    z = np.zeros((fld, K, Np))
    for j in range(n):
        z.flat[j] = 1.0
        d = O.rhs_full(O.State(z[0], list(z[1:])), od)
        A[:, j] = np.concatenate([a.ravel() for a in d.fields()])
        z.flat[j] = 0.0
    return A


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["tri", "tet"])
def test_device_matrix_matches_oracle(shape):
    mesh = meshgen.warped_triangle_mesh(2, 2) if shape == "tri" else meshgen.warped_cube_tet_mesh(1, 2)
    cfg = SolverConfig(N=2, formulation=Formulation.StrongWeak, flux=FluxParams(1.0, 1.0))
    A = an.assemble_evolution_matrix(mesh, cfg)
    B = oracle_matrix(mesh, 2, True, 1.0)
    assert A.shape == B.shape
    assert np.max(np.abs(A - B)) < 1e-11 * np.abs(B).max()


@pytest.mark.gpu
def test_linearity_and_size_cap(rng):
    from paper_1608_03836_b200 import solver
    mesh = meshgen.warped_triangle_mesh(2, 2)
    cfg = SolverConfig(N=2, flux=FluxParams(1, 1))
    A = an.assemble_evolution_matrix(mesh, cfg)
    disc = solver.Discretization(mesh, cfg)
    x = rng.standard_normal(A.shape[0])
    st = FieldState(*(x.reshape(3, mesh.K, disc.ref.Np)))
    d = solver.rhs_full(st, disc)
    direct = np.concatenate([np.asarray(a).ravel() for a in d.fields()])
    assert np.max(np.abs(A @ x - direct)) < 1e-12 * max(1, np.max(np.abs(direct)))
    with pytest.raises(an.SizeCapExceeded):
        an.assemble_evolution_matrix(mesh, cfg, cap=100)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", ["tri", "tet"])
def test_central_flux_skew_and_penalty_dissipative(shape):
    # curved triangles; affine tetrahedra (on curved tets the collapsed face rule is not
    # rotation symmetric, so the discrete energy identity holds only to quadrature accuracy)
    mesh = meshgen.warped_triangle_mesh(2, 3) if shape == "tri" else meshgen.warped_cube_tet_mesh(1, 2, amp=0.0)
    N = 3 if shape == "tri" else 2
    central = an.eigenspectrum(an.assemble_evolution_matrix(
        mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(0, 0))))
    assert central.max_real_part <= 1e-8 * central.spectral_radius
    lam = central.eigenvalues
    for v in lam[:40]:                                   # conjugate pairs
        assert np.min(np.abs(lam - np.conj(v))) < 1e-8 * central.spectral_radius
    pen = an.eigenspectrum(an.assemble_evolution_matrix(
        mesh, SolverConfig(N=N, formulation=Formulation.StrongWeak, flux=FluxParams(1, 1))))
    assert pen.max_real_part <= 1e-8 * pen.spectral_radius
    assert pen.eigenvalues.real.min() < -1e-6 * pen.spectral_radius


def test_replicate_mesh_copies_are_disjoint():
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    big = meshgen.replicate_mesh(mesh, 3)
    K = mesh.K
    assert big.K == 3 * K
    c = big.face_connectivity
    for k in range(big.K):
        for f in range(4):
            k2, f2 = c[k, f]
            if k2 >= 0:
                assert k2 // K == k // K and tuple(c[k2, f2]) == (k, f)
    assert np.array_equal(big.elem_map_nodes[2 * K:], mesh.elem_map_nodes)
    assert np.array_equal(big.face_orientation[K:2 * K], mesh.face_orientation)


@pytest.mark.gpu
def test_batched_assembly_equals_column_by_column():
    """Batches of columns on a replicated mesh give the same matrix bit for
    bit as one column per pass (same per-element arithmetic)."""
    mesh = meshgen.warped_cube_tet_mesh(1, 2)
    cfg = SolverConfig(N=2, formulation=Formulation.StrongWeak, flux=FluxParams(0.7, 1.3))
    A1 = an.assemble_evolution_matrix(mesh, cfg, batch=1)
    A7 = an.assemble_evolution_matrix(mesh, cfg, batch=7)
    Ad = an.assemble_evolution_matrix(mesh, cfg)
    assert np.array_equal(A1, A7) and np.array_equal(A1, Ad)
