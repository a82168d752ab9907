"""Reference element, geometry and mesh properties (2D restated from
R/pkg/tests/test_refelem.py / test_geometry.py, 3D generalised)."""

from fractions import Fraction
from math import comb, factorial

import numpy as np
import pytest

from paper_1608_03836_b200 import geometry, meshgen, refelem
from paper_1608_03836_b200.refelem import ElementShape

TET = ElementShape.Tetrahedron
TRI = ElementShape.Triangle
QUAD = ElementShape.Quadrilateral


def exact_tet_monomial(a, b, c):
    """int over the bi-unit tet of r^a s^b t^c, exact rational arithmetic."""
    tot = Fraction(0)
    for i in range(a + 1):
        for j in range(b + 1):
            for k in range(c + 1):
                coef = comb(a, i) * comb(b, j) * comb(c, k) * 2 ** (i + j + k) * (-1) ** (a - i + b - j + c - k)
                tot += Fraction(coef * factorial(i) * factorial(j) * factorial(k), factorial(i + j + k + 3))
    return float(8 * tot)


@pytest.mark.parametrize("degree", [0, 1, 3, 5, 7, 9, 11, 13, 15])
def test_tet_quadrature_exactness_and_positivity(degree):
    q = refelem.build_quadrature(TET, degree)
    assert np.all(q.weights > 0)
    assert q.weights.sum() == pytest.approx(4.0 / 3.0, rel=1e-14)
    for a in range(degree + 1):
        for b in range(degree + 1 - a):
            c = degree - a - b
            v = np.sum(q.weights * q.points[:, 0] ** a * q.points[:, 1] ** b * q.points[:, 2] ** c)
            assert v == pytest.approx(exact_tet_monomial(a, b, c), abs=1e-13)


@pytest.mark.parametrize("N", [1, 3, 5, 7])
def test_tet_basis_orthonormal_and_gradients(N):
    q = refelem.build_quadrature(TET, 2 * N + 2)
    V = refelem.eval_modal_basis(TET, N, q.points)
    G = V.T @ (q.weights[:, None] * V)
    assert np.max(np.abs(G - np.eye(len(G)))) < 1e-12
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 1, (400, 3))
    pts = pts[pts.sum(1) < -1.2][:15]
    grads = refelem.eval_modal_basis_grad(TET, N, pts)
    h = 1e-6
    for d in range(3):
        e = np.zeros(3)
        e[d] = h
        fd = (refelem.eval_modal_basis(TET, N, pts + e) - refelem.eval_modal_basis(TET, N, pts - e)) / (2 * h)
        assert np.max(np.abs(fd - grads[d])) < 1e-6 * max(1.0, np.abs(grads[d]).max())


@pytest.mark.parametrize("shape,N", [(TET, n) for n in range(1, 8)] + [(TRI, 4), (QUAD, 3)])
def test_reference_element_invariants(shape, N):
    ref = refelem.build_reference_element(N, shape)
    eye = np.eye(ref.Np)
    assert np.max(np.abs(ref.Pq @ ref.Vq - eye)) < 1e-12
    assert ref.cond_nodal < 100
    # reference derivatives are exact on the nodal interpolant of a degree-N polynomial
    x = ref.nodes
    xq = ref.volume_quad.points
    assert np.max(np.abs(ref.Drq @ x[:, 0] ** N - N * xq[:, 0] ** (N - 1))) < 1e-11
    # face traces from face nodes equal the full trace operator
    for f in range(ref.n_faces):
        blk = ref.Vfq[f * ref.nfq:(f + 1) * ref.nfq]
        assert np.max(np.abs(blk - ref.face_interp @ eye[ref.face_nodes[f]])) < 1e-12
    # the face node set is symmetric: every orientation is a permutation
    for perm in ref.face_perms:
        assert sorted(perm.tolist()) == list(range(ref.nfp))


@pytest.mark.parametrize("N", [2, 4])
def test_tet_face_nodes_lie_on_faces(N):
    ref = refelem.build_reference_element(N, TET)
    V = refelem.TET_VERTICES
    for f, (a, b, c) in enumerate(refelem.TET_FACE_VERTICES):
        n = np.cross(V[b] - V[a], V[c] - V[a])
        pts = ref.nodes[ref.face_nodes[f]]
        assert np.max(np.abs((pts - V[a]) @ n)) < 1e-12
        # outward orientation of the face parametrisation
        assert (V[a] - V.mean(axis=0)) @ n > 0


def test_triangle_nodes_carry_over_to_tet_faces():
    N = 5
    ref = refelem.build_reference_element(N, TET)
    tri = refelem.triangle_nodes(N)
    for f in range(4):
        pts = refelem.face_points(TET, f, tri)
        assert np.max(np.abs(ref.nodes[ref.face_nodes[f]] - pts)) < 1e-12


def test_cofactor_geometric_factors():
    mesh = meshgen.warped_cube_tet_mesh(2, 3)
    ref = refelem.build_reference_element(3, TET)
    g = geometry.compute_geometric_data(mesh, ref)
    # (dr/dx)(dx/dr) = I via the cofactor identity: check on x itself, d x_i / d x_j
    X = mesh.elem_map_nodes
    E = np.stack(refelem.nodal_grad_matrices(TET, 3, ref.volume_quad.points))
    jac = np.einsum("aqn,knd->kqda", E, X)            # dx_d / dr_a
    G = np.moveaxis(g.Gq, (0, 1), (2, 3))              # (K, Nq, a, i)
    prod = np.einsum("kqai,kqda->kqid", G, jac)
    assert np.max(np.abs(prod - np.eye(3))) < 1e-12


@pytest.mark.parametrize("N_geo", [1, 3])
def test_discrete_divergence_theorem_affine_tets(N_geo):
    mesh = meshgen.warped_cube_tet_mesh(3, N_geo, amp=0.0)
    ref = refelem.build_reference_element(3, TET)
    g = geometry.compute_geometric_data(mesh, ref)
    x, y, z = g.xyzq
    f = lambda x, y, z: x ** 2 * y + z ** 3 + x * y * z
    grad = [2 * x * y + y * z, x ** 2 + x * z, 3 * z ** 2 + x * y]
    xf, yf, zf = g.xyzfq
    for i in range(3):
        lhs = (ref.wq[None] * g.Jq * grad[i]).sum(1)
        rhs = (ref.wfq[None] * g.Jfq * g.nq[i] * f(xf, yf, zf)).sum(1)
        assert np.max(np.abs(lhs - rhs)) < 1e-12


def test_warped_cube_volume_and_boundary():
    mesh = meshgen.warped_cube_tet_mesh(4, 3)
    ref = refelem.build_reference_element(3, TET)
    g = geometry.compute_geometric_data(mesh, ref)
    assert geometry.element_areas(g).sum() == pytest.approx(8.0, rel=1e-10)
    assert g.Jq.min() > 0
    assert (mesh.boundary_tags > 0).sum() == 6 * 2 * 16
    # z-major: a z-layer of cubes is a contiguous element range
    nz_layer = 4 * 4 * 6
    zc = mesh.elem_map_nodes[:, :, 2].mean(axis=1)
    for L in range(4):
        layer = zc[L * nz_layer:(L + 1) * nz_layer]
        assert np.all((layer > -1 + 0.5 * L) & (layer < -1 + 0.5 * (L + 1)))


@pytest.mark.parametrize("make", [lambda: meshgen.warped_cube_tet_mesh(3, 2),
                                  lambda: meshgen.warped_triangle_mesh(4, 3),
                                  lambda: meshgen.uniform_quad_mesh(3, N_geo=2)])
def test_face_matching_by_orientation(make):
    """Neighbouring faces carry the same physical face nodes once permuted
    by the stored orientation code (the surface kernel's exterior gather)."""
    mesh = make()
    ref = refelem.build_reference_element(mesh.N_geo, mesh.shape)
    fm = np.array(ref.face_nodes)
    X = mesh.elem_map_nodes
    conn, ori = mesh.face_connectivity, mesh.face_orientation
    err = 0.0
    for k in range(mesh.K):
        for f in range(mesh.n_faces):
            k2, f2 = conn[k, f]
            if k2 < 0:
                continue
            assert tuple(conn[k2, f2]) == (k, f)
            mine = X[k, fm[f]]
            theirs = X[k2, fm[f2][ref.face_perms[ori[k, f]]]]
            err = max(err, np.abs(mine - theirs).max())
    assert err < 1e-12


def test_config1_mesh():
    mesh = meshgen.warped_triangle_mesh()
    assert mesh.K == 512 and mesh.N_geo == 4 and mesh.h == pytest.approx(0.125)
    ref = refelem.build_reference_element(4, TRI)
    g = geometry.compute_geometric_data(mesh, ref)
    assert g.Jq.min() > 0
    assert geometry.element_areas(g).sum() == pytest.approx(4.0, rel=1e-12)
    # the warp fixes the boundary of [-1, 1]^2
    xb = np.concatenate([g.xfq[mesh.boundary_tags.repeat(ref.nfq, axis=1) > 0]])
    yb = np.concatenate([g.yfq[mesh.boundary_tags.repeat(ref.nfq, axis=1) > 0]])
    on = (np.abs(np.abs(xb) - 1) < 1e-12) | (np.abs(np.abs(yb) - 1) < 1e-12)
    assert on.all()


def test_mesh_json_round_trip(tmp_path):
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    p = tmp_path / "m.json"
    meshgen.save_mesh(mesh, p)
    m2 = meshgen.load_mesh(p)
    assert m2.shape is TET and m2.K == mesh.K
    assert np.array_equal(m2.face_orientation, mesh.face_orientation)
    assert np.max(np.abs(m2.elem_map_nodes - mesh.elem_map_nodes)) == 0


@pytest.mark.parametrize("N,N_geo", [(2, 2), (3, 2), (3, 3), (4, 4)])
def test_discrete_divergence_theorem_curved_tets(N, N_geo, rng):
    """R/pkg/tests/test_geometry.py:116-137 transplanted to curved tets under
    the 3D sufficiency rules (volume 2N + 2N_geo - 3, face 2N + 2N_geo - 2):
    the volume quadrature of J div u equals the face quadrature of u.n sJ for
    random u in (P^N)^3, to 1e-10.  This pins the cofactor metric terms, the
    Nanson normals, sJ, the collapsed tet / triangle rules and the face
    parametrisation of the shared 3D setup independently of the solver."""
    import wadg_oracle as O
    mesh = meshgen.warped_cube_tet_mesh(2, N_geo)
    vdeg, fdeg = O.quadrature_degrees(N, N_geo, TET, False)
    ref = refelem.build_reference_element(N, TET, vdeg, fdeg)
    g = geometry.compute_geometric_data(mesh, ref)
    u = [rng.standard_normal((mesh.K, ref.Np)) for _ in range(3)]
    divJ = sum((u[i] @ ref.Dq[a].T) * (g.Gq[a, i] * g.Jq) for a in range(3) for i in range(3))
    vol = divJ @ ref.wq
    un = sum((u[i] @ ref.Vfq.T) * g.nq[i] for i in range(3))
    surf = (un * g.Jfq) @ ref.wfq
    assert np.max(np.abs(vol - surf)) < 1e-10
    # the warp is genuinely curved: with N_geo = 4 the default 2N+1 rules are below
    # the face degree N + 2 N_geo - 2 of u.n sJ, and the identity fails
    if N_geo >= 4:
        ref_lo = refelem.build_reference_element(N, TET, 2 * N + 1, 2 * N + 1)
        g_lo = geometry.compute_geometric_data(mesh, ref_lo)
        divJ = sum((u[i] @ ref_lo.Dq[a].T) * (g_lo.Gq[a, i] * g_lo.Jq) for a in range(3) for i in range(3))
        un = sum((u[i] @ ref_lo.Vfq.T) * g_lo.nq[i] for i in range(3))
        assert np.max(np.abs(divJ @ ref_lo.wq - (un * g_lo.Jfq) @ ref_lo.wfq)) > 1e-8


def test_tet_operators_exact_on_polynomials():
    """Reference tet operators against closed forms: Vq interpolates, Dq
    differentiates and Pq projects every monomial of total degree <= N exactly;
    the volume rule integrates r^a s^b t^c exactly up to its degree."""
    from math import factorial
    N = 4
    ref = refelem.build_reference_element(N, TET)
    r, s, t = ref.nodes.T
    rq, sq, tq = ref.volume_quad.points.T
    for a in range(N + 1):
        for b in range(N + 1 - a):
            for c in range(N + 1 - a - b):
                f = r ** a * s ** b * t ** c
                fq = rq ** a * sq ** b * tq ** c
                assert np.max(np.abs(ref.Vq @ f - fq)) < 1e-12
                d = [a * rq ** max(a - 1, 0) * sq ** b * tq ** c, b * rq ** a * sq ** max(b - 1, 0) * tq ** c,
                     c * rq ** a * sq ** b * tq ** max(c - 1, 0)]
                for k in range(3):
                    assert np.max(np.abs(ref.Dq[k] @ f - d[k])) < 1e-10
                assert np.max(np.abs(ref.Pq @ fq - f)) < 1e-11
    # exact integral over the bi-unit tet {r,s,t >= -1, r+s+t <= -1} of (1+r)^a (1+s)^b (1+t)^c
    # = 2^(a+b+c+3) a! b! c! / (a+b+c+3)!
    for a, b, c in [(0, 0, 0), (2, 1, 0), (3, 3, 3), (5, 2, 2)]:
        if a + b + c > 2 * N + 1:
            continue
        exact = 2.0 ** (a + b + c + 3) * factorial(a) * factorial(b) * factorial(c) / factorial(a + b + c + 3)
        got = ref.wq @ ((1 + rq) ** a * (1 + sq) ** b * (1 + tq) ** c)
        assert got == pytest.approx(exact, rel=1e-13)
