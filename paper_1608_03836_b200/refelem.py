"""Reference elements: quadrature rules, orthonormal modal bases, nodal sets
and the dense reference operators the device kernels consume.

Host-side setup (not on the timed path).  The 2D triangle / quadrilateral
constructions restate the reference package so that every matrix matches it
to rounding (pinned by ``tests/golden``):

* collapsed Duffy triangle rule ............ R/pkg/src/wadg/refelem.py:147-178
* Koornwinder-Dubiner / Legendre bases ..... R/pkg/src/wadg/refelem.py:198-249
* warped-equispaced triangle nodes ......... R/pkg/src/wadg/refelem.py:255-297
* operator assembly (Vq, Pq, Drq, Mhat ...)  R/pkg/src/wadg/refelem.py:400-453
* per-face node lists ...................... R/pkg/src/wadg/refelem.py:456-467

The tetrahedron is the 3D generalisation the reference does not ship
(SURVEY.md §8(c)): a Gauss-Legendre x Gauss-Jacobi(1,0) x Gauss-Jacobi(2,0)
collapsed rule, the orthonormal tetrahedral Dubiner basis, and an
equispaced-plus-edge-warp node set whose faces carry exactly the 2D triangle
node set (so neighbouring faces match by a vertex permutation).

Additions used by the device path (not in the reference):

* ``face_interp``  (nfq x nfp): face-node values -> face quadrature values,
  identical for every face because each face carries the same node set;
* ``face_perms``   (n_orient x nfp): face-node permutation for each relative
  orientation of two matching faces (2D: identity / reversal; 3D: the six
  vertex permutations).
"""

from __future__ import annotations

import enum
import itertools
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
from scipy import special as sps


class SingularNodalBasis(Exception):
    """Raised when an interpolation node set fails to be unisolvent."""


class ElementShape(enum.Enum):
    Triangle = "triangle"
    Quadrilateral = "quadrilateral"
    Tetrahedron = "tetrahedron"

    @property
    def dim(self):
        return 3 if self is ElementShape.Tetrahedron else 2

    @property
    def n_faces(self):
        return {"triangle": 3, "quadrilateral": 4, "tetrahedron": 4}[self.value]

    @property
    def n_vertices(self):
        return {"triangle": 3, "quadrilateral": 4, "tetrahedron": 4}[self.value]

    @property
    def measure(self):
        """Area / volume of the reference element."""
        return {"triangle": 2.0, "quadrilateral": 4.0, "tetrahedron": 4.0 / 3.0}[self.value]

    @property
    def face_shape(self):
        return ElementShape.Triangle if self is ElementShape.Tetrahedron else None


def basis_dimension(shape, N):
    if shape is ElementShape.Triangle:
        return (N + 1) * (N + 2) // 2
    if shape is ElementShape.Tetrahedron:
        return (N + 1) * (N + 2) * (N + 3) // 6
    return (N + 1) ** 2


# 2D faces: (midpoint, d(r,s)/dxi), counterclockwise (R/.../refelem.py:54-65).
_QUAD_FACES = (
    (np.array([0.0, -1.0]), np.array([1.0, 0.0])),
    (np.array([1.0, 0.0]), np.array([0.0, 1.0])),
    (np.array([0.0, 1.0]), np.array([-1.0, 0.0])),
    (np.array([-1.0, 0.0]), np.array([0.0, -1.0])),
)
_TRI_FACES = (
    (np.array([0.0, -1.0]), np.array([1.0, 0.0])),
    (np.array([0.0, 0.0]), np.array([-1.0, 1.0])),
    (np.array([-1.0, 0.0]), np.array([0.0, -1.0])),
)

# reference vertices; face vertex triples / pairs in face-parameter order
TRI_VERTICES = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])
QUAD_VERTICES = np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]])
TET_VERTICES = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0],
                         [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])
# face f is parametrised from its first vertex (xi = -1) toward the second
TRI_FACE_VERTICES = ((0, 1), (1, 2), (2, 0))
QUAD_FACE_VERTICES = ((0, 1), (1, 2), (2, 3), (3, 0))
# tet faces: t = -1, s = -1, r + s + t = -1, r = -1; each triple is ordered so
# that the face map (xi, eta) -> X has an outward (T_xi x T_eta)
TET_FACE_VERTICES = ((0, 2, 1), (0, 1, 3), (1, 2, 3), (0, 3, 2))


def face_vertices(shape):
    return {ElementShape.Triangle: TRI_FACE_VERTICES,
            ElementShape.Quadrilateral: QUAD_FACE_VERTICES,
            ElementShape.Tetrahedron: TET_FACE_VERTICES}[shape]


def reference_vertices(shape):
    return {ElementShape.Triangle: TRI_VERTICES,
            ElementShape.Quadrilateral: QUAD_VERTICES,
            ElementShape.Tetrahedron: TET_VERTICES}[shape]


def face_parametrizations(shape):
    """2D: per-face (midpoint, d(r,s)/dxi) pairs for xi in [-1, 1], CCW."""
    if shape is ElementShape.Tetrahedron:
        raise ValueError("tetrahedral faces are parametrised by face_points")
    return _TRI_FACES if shape is ElementShape.Triangle else _QUAD_FACES


def _tri_barycentric(xi, eta):
    """Barycentrics of (xi, eta) w.r.t. the reference triangle vertices."""
    return np.stack([-(xi + eta) / 2.0, (1.0 + xi) / 2.0, (1.0 + eta) / 2.0], axis=-1)


def face_points(shape, face, xi):
    """Map face parameters to reference coordinates on the given face.

    2D: xi is (n,) in [-1, 1].  3D: xi is (n, 2) points of the reference
    triangle, mapped through the face's ordered vertex triple."""
    if shape is ElementShape.Tetrahedron:
        xi = np.atleast_2d(np.asarray(xi, dtype=float))
        lam = _tri_barycentric(xi[:, 0], xi[:, 1])
        verts = TET_VERTICES[list(TET_FACE_VERTICES[face])]
        return lam @ verts
    mid, dvec = face_parametrizations(shape)[face]
    xi = np.asarray(xi, dtype=float)
    return mid[None, :] + xi[:, None] * dvec[None, :]


# ---------------------------------------------------------------------------
# 1D building blocks

@dataclass(frozen=True)
class QuadratureRule:
    """Points, positive weights, and the attained exactness degree."""

    points: np.ndarray
    weights: np.ndarray
    exactness_degree: int

    @property
    def n_points(self):
        return self.weights.shape[0]


def gauss_legendre_1d(n):
    if n < 1:
        raise ValueError(f"need at least one point, got n={n}")
    x, w = np.polynomial.legendre.leggauss(n)
    return QuadratureRule(points=x, weights=w, exactness_degree=2 * n - 1)


def gauss_lobatto_1d(n):
    if n < 2:
        raise ValueError(f"need at least two points, got n={n}")
    if n == 2:
        x = np.array([-1.0, 1.0])
    else:
        xi, _ = sps.roots_jacobi(n - 2, 1.0, 1.0)
        x = np.concatenate(([-1.0], np.sort(xi), [1.0]))
    pn = np.polynomial.legendre.Legendre.basis(n - 1)(x)
    w = 2.0 / (n * (n - 1) * pn ** 2)
    return QuadratureRule(points=x, weights=w, exactness_degree=2 * n - 3)


def jacobi_p(n, alpha, beta, x):
    """Orthonormal Jacobi polynomial: int P^2 (1-x)^a (1+x)^b dx = 1."""
    x = np.asarray(x, dtype=float)
    lg = sps.gammaln
    log_norm = ((alpha + beta + 1) * np.log(2.0) + lg(n + alpha + 1) + lg(n + beta + 1)
                - np.log(2 * n + alpha + beta + 1) - lg(n + 1) - lg(n + alpha + beta + 1))
    return sps.eval_jacobi(n, alpha, beta, x) / np.exp(0.5 * log_norm)


def grad_jacobi_p(n, alpha, beta, x, order=1):
    x = np.asarray(x, dtype=float)
    if order == 0:
        return jacobi_p(n, alpha, beta, x)
    coef = 1.0
    for k in range(order):
        if n - k <= 0:
            return np.zeros_like(x)
        coef *= np.sqrt((n - k) * (n + k + alpha + beta + 1))
    return coef * jacobi_p(n - order, alpha + order, beta + order, x)


# ---------------------------------------------------------------------------
# Volume quadrature

def _points_per_direction(degree):
    return max(1, (degree + 2) // 2)   # 2n - 1 >= degree


def build_quadrature(shape, degree):
    """Rule exact to (at least) ``degree``: tensor Gauss on the quad, and
    collapsed Gauss-Legendre x Gauss-Jacobi rules on simplices."""
    if degree < 0:
        raise ValueError(f"degree must be >= 0, got {degree}")
    n = _points_per_direction(degree)
    ga = gauss_legendre_1d(n)
    if shape is ElementShape.Quadrilateral:
        r, s = np.meshgrid(ga.points, ga.points, indexing="ij")
        return QuadratureRule(np.column_stack([r.ravel(), s.ravel()]),
                              np.outer(ga.weights, ga.weights).ravel(), 2 * n - 1)
    b, wb = sps.roots_jacobi(n, 1.0, 0.0)
    if shape is ElementShape.Triangle:
        A, B = np.meshgrid(ga.points, b, indexing="ij")
        r = 0.5 * (1 + A) * (1 - B) - 1
        return QuadratureRule(np.column_stack([r.ravel(), B.ravel()]),
                              (0.5 * np.outer(ga.weights, wb)).ravel(), 2 * n - 1)
    c, wc = sps.roots_jacobi(n, 2.0, 0.0)
    A, B, C = np.meshgrid(ga.points, b, c, indexing="ij")
    x, y = 0.5 * (1 - B), 0.5 * (1 - C)
    r = (1 + A) * x * y - 1
    s = (1 + B) * y - 1
    w = np.einsum("i,j,k->ijk", ga.weights, wb, wc) / 8.0
    return QuadratureRule(np.column_stack([r.ravel(), s.ravel(), C.ravel()]),
                          w.ravel(), 2 * n - 1)


# ---------------------------------------------------------------------------
# Orthonormal modal bases

def _modal_indices(shape, N):
    if shape is ElementShape.Triangle:
        return [(i, j) for i in range(N + 1) for j in range(N + 1 - i)]
    if shape is ElementShape.Tetrahedron:
        return [(i, j, k) for i in range(N + 1) for j in range(N + 1 - i)
                for k in range(N + 1 - i - j)]
    return [(i, j) for i in range(N + 1) for j in range(N + 1)]


def _pow(base, e):
    return base ** e if e >= 0 else np.zeros_like(base)


def _collapse_tri(r, s):
    a = np.full_like(r, -1.0)
    ok = s < 1.0 - 1e-14
    a[ok] = 2.0 * (1.0 + r[ok]) / (1.0 - s[ok]) - 1.0
    return a, s


def _collapse_tet(r, s, t):
    a = np.full_like(r, -1.0)
    ok = (s + t) < -1e-14
    a[ok] = 2.0 * (1.0 + r[ok]) / (-s[ok] - t[ok]) - 1.0
    b = np.full_like(r, -1.0)
    ok = t < 1.0 - 1e-14
    b[ok] = 2.0 * (1.0 + s[ok]) / (1.0 - t[ok]) - 1.0
    return a, b, t


def eval_modal_basis(shape, N, points):
    """Orthonormal basis values at ``points``, shape (n_points, Np)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    idx = _modal_indices(shape, N)
    V = np.empty((pts.shape[0], len(idx)))
    if shape is ElementShape.Quadrilateral:
        for m, (i, j) in enumerate(idx):
            V[:, m] = jacobi_p(i, 0, 0, pts[:, 0]) * jacobi_p(j, 0, 0, pts[:, 1])
        return V
    if shape is ElementShape.Triangle:
        a, b = _collapse_tri(pts[:, 0], pts[:, 1])
        x = 0.5 * (1.0 - b)
        for m, (i, j) in enumerate(idx):
            V[:, m] = (np.sqrt(2.0) * 2.0 ** i * jacobi_p(i, 0, 0, a)
                       * jacobi_p(j, 2 * i + 1, 0, b) * x ** i)
        return V
    a, b, c = _collapse_tet(pts[:, 0], pts[:, 1], pts[:, 2])
    x, y = 0.5 * (1.0 - b), 0.5 * (1.0 - c)
    for m, (i, j, k) in enumerate(idx):
        scale = 2.0 ** (0.5 * (4 * i + 2 * j + 3))
        V[:, m] = (scale * jacobi_p(i, 0, 0, a) * jacobi_p(j, 2 * i + 1, 0, b) * x ** i
                   * jacobi_p(k, 2 * i + 2 * j + 2, 0, c) * y ** (i + j))
    return V


def eval_modal_basis_grad(shape, N, points):
    """Reference-coordinate gradients of the orthonormal basis: a tuple of
    ``dim`` arrays (n_points, Np)."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    idx = _modal_indices(shape, N)
    grads = [np.empty((pts.shape[0], len(idx))) for _ in range(shape.dim)]
    if shape is ElementShape.Quadrilateral:
        r, s = pts[:, 0], pts[:, 1]
        for m, (i, j) in enumerate(idx):
            grads[0][:, m] = grad_jacobi_p(i, 0, 0, r) * jacobi_p(j, 0, 0, s)
            grads[1][:, m] = jacobi_p(i, 0, 0, r) * grad_jacobi_p(j, 0, 0, s)
        return tuple(grads)
    if shape is ElementShape.Triangle:
        a, b = _collapse_tri(pts[:, 0], pts[:, 1])
        x = 0.5 * (1.0 - b)
        for m, (i, j) in enumerate(idx):
            fa, dfa = jacobi_p(i, 0, 0, a), grad_jacobi_p(i, 0, 0, a)
            gb, dgb = jacobi_p(j, 2 * i + 1, 0, b), grad_jacobi_p(j, 2 * i + 1, 0, b)
            sc = np.sqrt(2.0) * 2.0 ** i
            xm1 = _pow(x, i - 1)
            grads[0][:, m] = sc * dfa * gb * xm1
            grads[1][:, m] = sc * (dfa * gb * 0.5 * (1.0 + a) * xm1
                                   + fa * (dgb * x ** i - 0.5 * i * gb * xm1))
        return tuple(grads)
    a, b, c = _collapse_tet(pts[:, 0], pts[:, 1], pts[:, 2])
    x, y = 0.5 * (1.0 - b), 0.5 * (1.0 - c)
    for m, (i, j, k) in enumerate(idx):
        sc = 2.0 ** (0.5 * (4 * i + 2 * j + 3))
        fa, dfa = jacobi_p(i, 0, 0, a), grad_jacobi_p(i, 0, 0, a)
        al = 2 * i + 1
        gb, dgb = jacobi_p(j, al, 0, b), grad_jacobi_p(j, al, 0, b)
        be = 2 * i + 2 * j + 2
        hc, dhc = jacobi_p(k, be, 0, c), grad_jacobi_p(k, be, 0, c)
        # psi = fa(a) * [gb x^i] * [hc y^(i+j)]
        ym1 = _pow(y, i + j - 1)
        d_r = dfa * gb * _pow(x, i - 1) * hc * ym1
        g_b = dgb * x ** i - 0.5 * i * gb * _pow(x, i - 1)       # d/db of gb x^i
        h_c = dhc * y ** (i + j) - 0.5 * (i + j) * hc * ym1       # d/dc of hc y^(i+j)
        tail = fa * g_b * hc * ym1
        grads[0][:, m] = sc * d_r
        grads[1][:, m] = sc * (0.5 * (1.0 + a) * d_r + tail)
        grads[2][:, m] = sc * (0.5 * (1.0 + a) * d_r + 0.5 * (1.0 + b) * tail
                               + fa * gb * x ** i * h_c)
    return tuple(grads)


# ---------------------------------------------------------------------------
# Interpolation nodes

def _warp_factor_1d(N, r):
    """Displacement pulling equispaced points onto Gauss-Lobatto points."""
    req = np.linspace(-1.0, 1.0, N + 1)
    gll = gauss_lobatto_1d(N + 1).points
    coeffs = np.linalg.solve(np.vander(req, increasing=True), gll - req)
    return np.vander(np.asarray(r), N + 1, increasing=True) @ coeffs


def _simplex_nodes(N, verts, lam):
    """Equispaced barycentric points warped edge by edge toward GLL points,
    blended into the interior (the reference's triangle construction,
    R/.../refelem.py:275-297, applied to every simplex edge)."""
    nodes = lam @ verts
    nv = verts.shape[0]
    edges = ((0, 1), (1, 2), (2, 0)) if nv == 3 else tuple(itertools.combinations(range(nv), 2))
    for i, j in edges:
        xi = lam[:, j] - lam[:, i]
        warp = _warp_factor_1d(N, xi)
        sf = 1.0 - xi ** 2
        blend = 4.0 * lam[:, i] * lam[:, j]
        ok = sf > 1e-12
        scale = np.zeros(len(lam))
        scale[ok] = blend[ok] / sf[ok]
        nodes = nodes + (scale * warp)[:, None] * 0.5 * (verts[j] - verts[i])[None, :]
    return nodes


def triangle_barycentric_lattice(N):
    lam = []
    for i in range(N + 1):
        for j in range(N + 1 - i):
            l2, l3 = i / N, j / N
            lam.append((1.0 - l2 - l3, l2, l3))
    return np.array(lam)


def triangle_nodes(N):
    if N < 1:
        raise ValueError("N must be >= 1")
    return _simplex_nodes(N, TRI_VERTICES, triangle_barycentric_lattice(N))


def tet_nodes(N):
    """Boundary-including tetrahedral node set; every face carries the 2D
    triangle node set (edge warps with a zero blend off the face)."""
    if N < 1:
        raise ValueError("N must be >= 1")
    lam = []
    for i in range(N + 1):
        for j in range(N + 1 - i):
            for k in range(N + 1 - i - j):
                l1, l2, l3 = i / N, j / N, k / N
                lam.append((1.0 - l1 - l2 - l3, l1, l2, l3))
    return _simplex_nodes(N, TET_VERTICES, np.array(lam))


def quad_nodes(N):
    if N < 1:
        raise ValueError("N must be >= 1")
    g = gauss_lobatto_1d(N + 1).points
    r, s = np.meshgrid(g, g, indexing="xy")
    return np.column_stack([r.ravel(), s.ravel()])


def interpolation_nodes(shape, N):
    if shape is ElementShape.Quadrilateral:
        return quad_nodes(N)
    if shape is ElementShape.Tetrahedron:
        return tet_nodes(N)
    return triangle_nodes(N)


def nodal_vandermonde(shape, N, nodes):
    V = eval_modal_basis(shape, N, nodes)
    if V.shape[0] != V.shape[1]:
        raise SingularNodalBasis(
            f"{V.shape[0]} nodes cannot be unisolvent for dimension {V.shape[1]}")
    cond = np.linalg.cond(V)
    if not np.isfinite(cond) or cond > 1e12:
        raise SingularNodalBasis(f"nodal basis condition number {cond:.3e}")
    return V, cond


@lru_cache(maxsize=None)
def _cached_nodal_basis(shape, N):
    nodes = interpolation_nodes(shape, N)
    V, cond = nodal_vandermonde(shape, N, nodes)
    return nodes, V, cond


def nodal_eval_matrix(shape, N, points):
    _, V, _ = _cached_nodal_basis(shape, N)
    return np.linalg.solve(V.T, eval_modal_basis(shape, N, points).T).T


def nodal_grad_matrices(shape, N, points):
    _, V, _ = _cached_nodal_basis(shape, N)
    return tuple(np.linalg.solve(V.T, G.T).T for G in eval_modal_basis_grad(shape, N, points))


# ---------------------------------------------------------------------------
# Reference element

@dataclass
class ReferenceElement:
    """Degree-N operator data on one reference shape (read-only once built)."""

    N: int
    shape: ElementShape
    nodes: np.ndarray
    volume_quad: QuadratureRule
    Vq: np.ndarray             # (Nq, Np)
    Pq: np.ndarray             # (Np, Nq) = Mhat^-1 Vq^T W
    Dq: tuple                  # dim x (Nq, Np) reference derivatives at quad points
    Mhat: np.ndarray
    Mhat_inv: np.ndarray
    face_quad: QuadratureRule  # rule on one face (1D Gauss in 2D, collapsed tri in 3D)
    face_nodes: list = field(repr=False)   # per-face volume-node indices (nfp each)
    Vfq: np.ndarray = field(repr=False)    # (n_faces*nfq, Np)
    Pfq: np.ndarray = field(repr=False)    # (Np, n_faces*nfq)
    wfq: np.ndarray = field(repr=False)
    face_quad_points: np.ndarray = field(repr=False)
    face_interp: np.ndarray = field(repr=False)   # (nfq, nfp)
    face_perms: np.ndarray = field(repr=False)    # (n_orient, nfp)
    cond_nodal: float = 0.0

    @property
    def Np(self):
        return self.nodes.shape[0]

    @property
    def Nq(self):
        return self.volume_quad.n_points

    @property
    def n_faces(self):
        return self.shape.n_faces

    @property
    def nfq(self):
        return self.face_quad.n_points

    @property
    def nfp(self):
        return len(self.face_nodes[0])

    @property
    def dim(self):
        return self.shape.dim

    @property
    def wq(self):
        return self.volume_quad.weights

    # reference-compatible names
    @property
    def Drq(self):
        return self.Dq[0]

    @property
    def Dsq(self):
        return self.Dq[1]

    @property
    def Dtq(self):
        return self.Dq[2] if self.dim == 3 else None

    @property
    def face_quad_1d(self):
        return self.face_quad


def face_rule(shape, degree):
    if shape is ElementShape.Tetrahedron:
        return build_quadrature(ElementShape.Triangle, degree)
    return gauss_legendre_1d(_points_per_direction(degree))


def _face_node_param(shape, N):
    """Face-node positions in the face parameter (the order face_nodes uses)."""
    if shape is ElementShape.Tetrahedron:
        return triangle_nodes(N)
    if shape is ElementShape.Quadrilateral:
        return gauss_lobatto_1d(N + 1).points
    # triangle edges carry the warped equispaced edge nodes = GLL points
    return gauss_lobatto_1d(N + 1).points


def _face_node_indices(shape, nodes, N, tol=1e-10):
    out = []
    if shape is ElementShape.Tetrahedron:
        par = _face_node_param(shape, N)
        for f in range(shape.n_faces):
            pts = face_points(shape, f, par)
            d = np.linalg.norm(nodes[None, :, :] - pts[:, None, :], axis=2)
            idx = np.argmin(d, axis=1)
            if np.max(d[np.arange(len(idx)), idx]) > 1e-9:
                raise SingularNodalBasis("tet face nodes do not match the triangle node set")
            out.append(idx)
        return out
    for f in range(shape.n_faces):
        mid, dvec = face_parametrizations(shape)[f]
        rel = nodes - mid[None, :]
        perp = np.abs(rel[:, 0] * dvec[1] - rel[:, 1] * dvec[0])
        xi = (rel @ dvec) / (dvec @ dvec)
        on = np.where((perp < tol) & (xi > -1 - tol) & (xi < 1 + tol))[0]
        out.append(on[np.argsort(xi[on])])
    return out


def orientation_permutations(shape):
    """Vertex permutations pi of one face: code c -> pi with pi[n] = m meaning
    neighbour-face vertex n is my face vertex m."""
    nv = 3 if shape is ElementShape.Tetrahedron else 2
    return [tuple(p) for p in itertools.permutations(range(nv))]


def _face_barycentric(shape, N):
    par = _face_node_param(shape, N)
    if shape is ElementShape.Tetrahedron:
        return _tri_barycentric(par[:, 0], par[:, 1])
    return np.stack([(1.0 - par) / 2.0, (1.0 + par) / 2.0], axis=-1)


def build_face_perms(shape, N):
    """perm[c][i] = neighbour face-node index of the point at my face node i
    when the faces meet with relative orientation code c."""
    bary = _face_barycentric(shape, N)
    perms = []
    for pi in orientation_permutations(shape):
        target = bary[:, list(pi)]            # nu_n = mu_{pi(n)}
        d = np.linalg.norm(bary[None, :, :] - target[:, None, :], axis=2)
        j = np.argmin(d, axis=1)
        if np.max(d[np.arange(len(j)), j]) > 1e-10:
            raise SingularNodalBasis("face node set is not symmetric")
        perms.append(j)
    return np.array(perms, dtype=np.int64)


def build_reference_element(N, shape, volume_quad_degree=None, face_quad_degree=None):
    """Assemble a ReferenceElement; defaults to degree-(2N+1) rules and floors
    the volume rule at 2N (R/.../refelem.py:400-453)."""
    if N < 1:
        raise ValueError("N must be >= 1")
    if volume_quad_degree is None:
        volume_quad_degree = 2 * N + 1
    if face_quad_degree is None:
        face_quad_degree = 2 * N + 1
    volume_quad_degree = max(volume_quad_degree, 2 * N)

    nodes, Vmodal, cond = _cached_nodal_basis(shape, N)
    quad = build_quadrature(shape, volume_quad_degree)

    def to_nodal(M):
        return np.linalg.solve(Vmodal.T, M.T).T

    Vq = to_nodal(eval_modal_basis(shape, N, quad.points))
    Dq = tuple(to_nodal(G) for G in eval_modal_basis_grad(shape, N, quad.points))
    wq = quad.weights
    Mhat = Vq.T @ (wq[:, None] * Vq)
    Mhat = 0.5 * (Mhat + Mhat.T)
    Mhat_inv = np.linalg.inv(Mhat)
    Pq = Mhat_inv @ (Vq.T * wq[None, :])

    frule = face_rule(shape, face_quad_degree)
    fq_pts, Vf_blocks, wf_blocks = [], [], []
    for f in range(shape.n_faces):
        pts = face_points(shape, f, frule.points)
        fq_pts.append(pts)
        Vf_blocks.append(to_nodal(eval_modal_basis(shape, N, pts)))
        wf_blocks.append(frule.weights)
    Vfq = np.vstack(Vf_blocks)
    wfq = np.concatenate(wf_blocks)
    Pfq = Mhat_inv @ (Vfq.T * wfq[None, :])

    face_nodes = _face_node_indices(shape, nodes, N)
    if shape is ElementShape.Tetrahedron:
        face_interp = nodal_eval_matrix(ElementShape.Triangle, N, frule.points)
    else:
        gl = _face_node_param(shape, N)
        L = np.polynomial.legendre.legvander
        face_interp = np.linalg.solve(L(gl, N).T, L(frule.points, N).T).T

    ref = ReferenceElement(
        N=N, shape=shape, nodes=nodes, volume_quad=quad, Vq=Vq, Pq=Pq, Dq=Dq,
        Mhat=Mhat, Mhat_inv=Mhat_inv, face_quad=frule, face_nodes=face_nodes,
        Vfq=Vfq, Pfq=Pfq, wfq=wfq, face_quad_points=np.vstack(fq_pts),
        face_interp=face_interp, face_perms=build_face_perms(shape, N), cond_nodal=cond)
    _validate_reference_element(ref)
    return ref


def _validate_reference_element(ref):
    Np = ref.Np
    if Np != basis_dimension(ref.shape, ref.N):
        raise SingularNodalBasis("node count does not match basis dimension")
    eye = np.eye(Np)
    if np.max(np.abs(ref.Pq @ ref.Vq - eye)) > 1e-10:
        raise FloatingPointError("Pq Vq deviates from identity")
    if np.max(np.abs(ref.Mhat_inv @ ref.Mhat - eye)) > 1e-10:
        raise FloatingPointError("Mhat inverse inaccurate")
    np.linalg.cholesky(ref.Mhat)
