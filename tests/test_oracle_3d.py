"""3D oracle pins.  The reference ships no 3D solver (R/SPEC.md:14-15), so
the tetrahedral branch of the oracle is pinned by the reference's own solver
invariants (R/pkg/tests/test_solver.py) transplanted to 3D, the exact LSRK
amplification polynomial and convergence to the exact Dirichlet eigenmode of
the cube (the configs' initial condition)."""

from fractions import Fraction

import numpy as np
import pytest

import wadg_oracle as O
from paper_1608_03836_b200 import meshgen, refelem
from paper_1608_03836_b200.refelem import ElementShape

TET = ElementShape.Tetrahedron


def rand_state(od, rng, K):
    return O.State(rng.standard_normal((K, od.ref.Np)), [rng.standard_normal((K, od.ref.Np)) for _ in range(3)])


def energy_rate(st, od):
    """d/dt of the quadratic energy from the premultiplied RHS
    (R/pkg/tests/test_solver.py:24-30)."""
    pre = O.rhs_pre_mass(st, od)
    Mh = od.ref.Mhat
    return sum(np.einsum("ki,ij,kj->", a, Mh, b) for a, b in zip(st.fields(), pre.fields()))


def single_curved_tet(N_geo=2):
    nodes = refelem.tet_nodes(N_geo)
    r, s, t = nodes.T
    X = np.stack([r + 0.08 * r * s, s - 0.06 * s * t * r, t + 0.05 * r ** 2], axis=1)[None]
    return meshgen.CurvedMesh(TET, N_geo, X, np.full((1, 4, 2), -1, dtype=np.int64),
                              np.ones((1, 4), dtype=np.int64), h=2.0,
                              face_orientation=np.zeros((1, 4), dtype=np.int64))


def test_constant_state_interior_rhs_zero():
    mesh = meshgen.warped_cube_tet_mesh(3, 2)
    for sw in (True, False):
        od = O.OracleDiscretization(mesh, 2, sw)
        K, Np = mesh.K, od.ref.Np
        st = O.State(np.full((K, Np), 3.14), [np.zeros((K, Np)) for _ in range(3)])
        d = O.rhs_pre_mass(st, od)
        interior = ~mesh.boundary_tags.any(axis=1)
        assert interior.sum() > 0
        for arr in d.fields():
            assert np.max(np.abs(arr[interior])) < 1e-11


def test_strong_equals_strong_weak_with_sufficient_quadrature(rng):
    N, mesh = 2, meshgen.warped_cube_tet_mesh(2, 2)
    vdeg, fdeg = O.quadrature_degrees(N, mesh.N_geo, TET, False)
    dS = O.OracleDiscretization(mesh, N, False)
    dW = O.OracleDiscretization(mesh, N, True, vol_deg=vdeg, face_deg=fdeg)
    for _ in range(3):
        st = rand_state(dS, rng, mesh.K)
        a, b = O.rhs_pre_mass(st, dS), O.rhs_pre_mass(st, dW)
        for x, y in zip(a.fields(), b.fields()):
            assert np.max(np.abs(x - y)) < 1e-9 * max(1.0, np.abs(y).max())


def test_single_curved_element_energy_rate_zero(rng):
    mesh = single_curved_tet()
    od = O.OracleDiscretization(mesh, 3, False, 0.0, 0.0)
    st = rand_state(od, rng, 1)
    assert abs(energy_rate(st, od)) < 1e-10


@pytest.mark.parametrize("curved", [False, True])
def test_energy_rate_equals_face_jump_dissipation(rng, curved):
    """dE/dt = -1/4 sum w sJ (tau_p [p]^2 + tau_u [u.n]^2)
    (R/pkg/tests/test_solver.py:80-105).  The central flux terms of the two
    sides of a face telescope only if both sides integrate with the same
    points; the collapsed triangle face rule is not rotation-symmetric, so on
    curved faces (sJ n non-constant) the identity holds to quadrature
    accuracy, and to rounding on affine faces."""
    tau_p, tau_u = 0.7, 1.3
    mesh = meshgen.warped_cube_tet_mesh(2, 2, amp=0.1 if curved else 0.0)
    od = O.OracleDiscretization(mesh, 3, True, tau_p, tau_u)
    st = rand_state(od, rng, mesh.K)
    dE = energy_rate(st, od)
    bc = od.bc_mask
    pM, pP = od.face_traces(st.p)
    uM, uP = zip(*[od.face_traces(a) for a in st.u])
    pP = np.where(bc, -pM, pP)
    uP = [np.where(bc, a, b) for a, b in zip(uM, uP)]
    n = od.geo.nq
    dp = pP - pM
    dun = sum((uP[i] - uM[i]) * n[i] for i in range(3))
    quad = np.sum(od.ref.wfq[None, :] * od.geo.Jfq * (tau_p * dp ** 2 + tau_u * dun ** 2))
    assert dE == pytest.approx(-0.25 * quad, rel=1e-3 if curved else 1e-10)
    assert dE < 0


def test_energy_rate_identity_curved_tets_sufficient_quadrature(rng):
    """R/pkg/tests/test_solver.py:80-105 on curved tets, split by what is
    exact.  With the strong-form sufficiency rules (volume 2N + 2N_geo - 3,
    face 2N + 2N_geo - 2):
    * tau = 0: the central-flux terms telescope exactly although the two
      sides of a face integrate at different collapsed-rule points, because
      p u.(n sJ) is a polynomial the face rule integrates exactly on both
      sides (n sJ is the polynomial Nanson area vector): dE/dt = 0 to rounding;
    * tau > 0: the penalty terms carry sJ = |n sJ| and n = (n sJ)/sJ, which are
      not polynomials on curved faces, so the identity holds to the face
      rule's accuracy (1e-6 measured; 1e-3 with the default 2N+1 rule)."""
    N = 3
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    vdeg, fdeg = O.quadrature_degrees(N, mesh.N_geo, TET, False)
    od0 = O.OracleDiscretization(mesh, N, True, 0.0, 0.0, vol_deg=vdeg, face_deg=fdeg)
    st = rand_state(od0, rng, mesh.K)
    scale = sum(float(np.abs(a).sum()) for a in st.fields())
    assert abs(energy_rate(st, od0)) < 1e-14 * scale
    tau_p, tau_u = 0.7, 1.3
    od = O.OracleDiscretization(mesh, N, True, tau_p, tau_u, vol_deg=vdeg, face_deg=fdeg)
    dE = energy_rate(st, od)
    bc = od.bc_mask
    pM, pP = od.face_traces(st.p)
    uM, uP = zip(*[od.face_traces(a) for a in st.u])
    pP = np.where(bc, -pM, pP)
    uP = [np.where(bc, a, b) for a, b in zip(uM, uP)]
    n = od.geo.nq
    dun = sum((uP[i] - uM[i]) * n[i] for i in range(3))
    quad = np.sum(od.ref.wfq[None, :] * od.geo.Jfq * (tau_p * (pP - pM) ** 2 + tau_u * dun ** 2))
    assert dE == pytest.approx(-0.25 * quad, rel=1e-5)
    assert dE < 0


def test_wadg_exact_on_affine_elements(rng):
    """J constant per element: Pq diag(1/J) Vq r == r / J (the exact mass
    inverse), for both fields (c^2 = 1)."""
    mesh = meshgen.warped_cube_tet_mesh(2, 1, amp=0.0)
    od = O.OracleDiscretization(mesh, 3, True)
    st = rand_state(od, rng, mesh.K)
    out = O.apply_mass_inverse(st, od)
    J = 1.0 / od.w_upd_u[:, :1]
    for a, b in zip(out.fields(), st.fields()):
        assert np.max(np.abs(a - b / J)) < 1e-10 * np.abs(b / J).max()


def test_pointwise_heterogeneous_weights():
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(2, 2)
    od = O.OracleDiscretization(mesh, 2, True, c2=c2)
    from paper_1608_03836_b200 import geometry
    gu = geometry.compute_geometric_data(mesh, od.ref_upd)
    assert np.max(np.abs(od.w_upd_p - c2(*gu.xyzq) / gu.Jq)) < 1e-14


def test_lsrk_amplification_polynomial():
    """Exact rational recurrence of the coefficient set (R/pkg/tests/test_solver.py:156-187)."""
    A = [Fraction(0), Fraction(-567301805773, 1357537059087), Fraction(-2404267990393, 2016746695238),
         Fraction(-3550918686646, 2091501179385), Fraction(-1275806237668, 842570457699)]
    B = [Fraction(1432997174477, 9575080441755), Fraction(5161836677717, 13612068292357),
         Fraction(1720146321549, 2090206949498), Fraction(3134564353537, 4481467310338),
         Fraction(2277821191437, 14882151754819)]
    yp, rp = [Fraction(1)], [Fraction(0)]

    def add(p, q):
        n = max(len(p), len(q))
        return [(p[i] if i < len(p) else 0) + (q[i] if i < len(q) else 0) for i in range(n)]

    for a, b in zip(A, B):
        rp = add([a * c for c in rp], [Fraction(0)] + yp)
        yp = add(yp, [b * c for c in rp])
    R = [float(c) for c in yp]
    assert R[:5] == pytest.approx([1, 1, 0.5, 1 / 6, 1 / 24], abs=1e-15)
    lam, dt = -0.37, 0.21
    st = O.State(np.array([[1.0]]), [np.zeros((1, 1))] * 3)
    out = O.lsrk_step(st, dt, lambda s: O.State(lam * s.p, [0 * a for a in s.u]))
    assert out.p[0, 0] == pytest.approx(sum(c * (lam * dt) ** k for k, c in enumerate(R)), abs=1e-14)


def test_dirichlet_eigenmode_convergence():
    """The configs' IC p = prod cos(pi x_i / 2), u = 0 is the lowest
    Dirichlet mode: p = cos(w t) prod cos(pi x_i / 2), w = pi sqrt(3) / 2."""
    N, T = 2, 0.2
    w = np.pi * np.sqrt(3) / 2
    phi = lambda x, y, z: np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * z / 2)
    errs, hs = [], []
    for n in (2, 4):
        mesh = meshgen.warped_cube_tet_mesh(n, N)
        od = O.OracleDiscretization(mesh, N, True)
        st = O.project_initial_condition(mesh, N, lambda x, y, z: (phi(x, y, z),) + (0 * x,) * 3)
        steps = int(np.ceil(T / (0.5 * (2 / n) / (N + 1) ** 2)))
        dt = T / steps
        for _ in range(steps):
            st = O.lsrk_step(st, dt, lambda y: O.rhs_full(y, od))
        ref_e = refelem.build_reference_element(N, TET, 2 * N + 4, 1)
        from paper_1608_03836_b200 import geometry
        ge = geometry.compute_geometric_data(mesh, ref_e)
        uq = st.p @ ref_e.Vq.T
        err = np.sqrt(np.sum(ref_e.wq[None] * ge.Jq * (uq - np.cos(w * T) * phi(*ge.xyzq)) ** 2))
        errs.append(err)
        hs.append(2 / n)
    slope = np.log(errs[0] / errs[1]) / np.log(hs[0] / hs[1])
    assert slope > N + 0.5


def test_wadg_and_exact_mass_errors_agree_on_curved_tets():
    """The paper's accuracy claim in 3D (analogue of R/pkg/tests/test_solver.py:
    143-152): against the exact Dirichlet eigenmode, WADG and the dense
    ExactCurvedMass inverse give the same error to within 1 %."""
    N, n, T, steps = 2, 3, 0.2, 10
    mesh = meshgen.warped_cube_tet_mesh(n, N)
    w = np.pi * np.sqrt(3) / 2

    def ic(x, y, z):
        p = np.cos(np.pi * x / 2) * np.cos(np.pi * y / 2) * np.cos(np.pi * z / 2)
        return p, 0 * p, 0 * p, 0 * p

    errs = []
    for exact in (False, True):
        od = O.OracleDiscretization(mesh, N, True, exact_mass=exact)
        st = O.project_initial_condition(mesh, N, ic)
        for _ in range(steps):
            st = O.lsrk_step(st, T / steps, lambda y: O.rhs_full(y, od))
        xq = od.geo.xyzq
        pex = np.cos(np.pi * xq[0] / 2) * np.cos(np.pi * xq[1] / 2) * np.cos(np.pi * xq[2] / 2) * np.cos(w * T)
        W = od.ref.wq[None, :] * od.geo.Jq
        errs.append(np.sqrt(np.sum(W * (od.interp(st.p) - pex) ** 2)))
    assert 0.99 <= errs[0] / errs[1] <= 1.01


def test_submesh_patch_reproduces_element_rhs(rng):
    """The helper behind the full-size sampled GPU parity test: the oracle
    RHS of an element computed on its one-neighbour patch equals the RHS on
    the whole mesh (heterogeneous medium, curved tets)."""
    from conftest import submesh
    c2 = lambda x, y, z: 1 + 0.5 * np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)
    mesh = meshgen.warped_cube_tet_mesh(4, 2)
    od = O.OracleDiscretization(mesh, 2, True, 0.7, 1.3, c2=c2)
    st = rand_state(od, rng, mesh.K)
    full = O.rhs_full(st, od).fields()
    elems = np.array([0, 7, 100, 200, mesh.K - 1])
    sub, patch, loc = submesh(mesh, elems)
    assert sub.K < mesh.K
    osub = O.OracleDiscretization(sub, 2, True, 0.7, 1.3, c2=c2)
    part = O.rhs_full(O.State(st.p[patch], [a[patch] for a in st.u]), osub).fields()
    for x, y in zip(part, full):
        assert np.max(np.abs(x[loc] - y[elems])) < 1e-12 * np.abs(y).max()
