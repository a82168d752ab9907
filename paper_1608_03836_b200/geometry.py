"""Isoparametric map evaluation: Jacobians, scaled geometric factors, face
normals and surface Jacobians at quadrature points (host/device setup).

Follows R/pkg/src/wadg/geometry.py:56-102 in 2D (J = x_r y_s - x_s y_r,
r_x = y_s / J ..., outward normal (y', -x') / sJ along the CCW face
parameter); in 3D the scaled factors are the cofactors of dx/dr and the face
normal is the cross product of the two face-parameter tangents (Nanson).

The core works on torch float64 tensors so the same code runs on the host for
small meshes (numpy views for the reference-compatible API) and in element
chunks on the GPU for million-element meshes, writing straight into the
device layout.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import refelem
from .refelem import ElementShape


class NonPositiveJacobian(Exception):
    """Mapping Jacobian fails to be positive at a checked point."""

    def __init__(self, element, point, value):
        self.element = element
        self.point = point
        self.value = value
        super().__init__(
            f"J = {value:.3e} <= 0 on element {element} at quadrature point {point}")


@dataclass
class GeometricData:
    """Per-element metric data at the quadrature points of one reference
    element.  Volume arrays are (K, Nq); face arrays (K, n_faces * nfq)."""

    ref: refelem.ReferenceElement = field(repr=False)
    xyzq: tuple = field(repr=False)       # dim arrays of physical coordinates
    Jq: np.ndarray = field(repr=False)
    Gq: np.ndarray = field(repr=False)    # (dim, dim, K, Nq): d r_a / d x_i
    xyzfq: tuple = field(repr=False)
    Jfq: np.ndarray = field(repr=False)   # surface Jacobian per face parameter measure
    nq: tuple = field(repr=False)         # dim arrays of unit outward normals

    @property
    def K(self):
        return self.Jq.shape[0]

    # reference-compatible names (2D: R/.../geometry.py:31-49)
    @property
    def xq(self):
        return self.xyzq[0]

    @property
    def yq(self):
        return self.xyzq[1]

    @property
    def zq(self):
        return self.xyzq[2]

    @property
    def rxq(self):
        return self.Gq[0, 0]

    @property
    def ryq(self):
        return self.Gq[0, 1]

    @property
    def sxq(self):
        return self.Gq[1, 0]

    @property
    def syq(self):
        return self.Gq[1, 1]

    @property
    def xfq(self):
        return self.xyzfq[0]

    @property
    def yfq(self):
        return self.xyzfq[1]

    @property
    def zfq(self):
        return self.xyzfq[2]

    @property
    def nxq(self):
        return self.nq[0]

    @property
    def nyq(self):
        return self.nq[1]

    @property
    def nzq(self):
        return self.nq[2]


@dataclass
class MapOperators:
    """Map-node evaluation matrices at the volume and face quadrature points
    of one reference element (host numpy, converted per device on demand)."""

    E: np.ndarray      # (Nq, Npg)
    Eg: np.ndarray     # (dim, Nq, Npg)
    Ef: np.ndarray     # (nf*nfq, Npg)
    Efg: np.ndarray    # (dim, nf*nfq, Npg)
    tangents: np.ndarray   # (nf, dim-1, dim) reference face tangent vectors
    nfq: int

    def to(self, device):
        t = lambda a: torch.as_tensor(a, dtype=torch.float64, device=device)
        return {"E": t(self.E), "Eg": t(self.Eg), "Ef": t(self.Ef), "Efg": t(self.Efg),
                "tangents": t(self.tangents)}


def map_operators(shape, N_geo, ref):
    E = refelem.nodal_eval_matrix(shape, N_geo, ref.volume_quad.points)
    Eg = np.stack(refelem.nodal_grad_matrices(shape, N_geo, ref.volume_quad.points))
    Ef = refelem.nodal_eval_matrix(shape, N_geo, ref.face_quad_points)
    Efg = np.stack(refelem.nodal_grad_matrices(shape, N_geo, ref.face_quad_points))
    if shape is ElementShape.Tetrahedron:
        V = refelem.TET_VERTICES
        tang = np.array([[0.5 * (V[b] - V[a]), 0.5 * (V[c] - V[a])]
                         for a, b, c in refelem.TET_FACE_VERTICES])
    else:
        tang = np.array([[d] for _, d in refelem.face_parametrizations(shape)])
    return MapOperators(E, Eg, Ef, Efg, tang, ref.nfq)


def geometric_factors(X, mops, check=True, k_offset=0):
    """Metric data of a chunk of elements.

    X: (Kc, Npg, dim) float64 tensor of map-node coordinates; mops: dict from
    MapOperators.to(device).  Returns a dict of tensors:
      xq (dim, Kc, Nq), J (Kc, Nq), GJ (dim, dim, Kc, Nq) = (dr_a/dx_i) J,
      xf (dim, Kc, F), sJ (Kc, F), n (dim, Kc, F)  with F = nf * nfq.
    """
    dim = X.shape[2]
    xq = torch.einsum("qn,knd->dkq", mops["E"], X)
    jac = torch.einsum("aqn,knd->dakq", mops["Eg"], X)      # jac[d, a] = dx_d / dr_a
    if dim == 2:
        J = jac[0, 0] * jac[1, 1] - jac[0, 1] * jac[1, 0]
        GJ = torch.stack([torch.stack([jac[1, 1], -jac[0, 1]]),
                          torch.stack([-jac[1, 0], jac[0, 0]])])
    else:
        cof = lambda a, b, c, d: jac[a, b] * jac[c, d] - jac[a, d] * jac[c, b]
        # adj[a, i] = cofactor(i, a) of jac: (dr_a/dx_i) J
        GJ = torch.stack([
            torch.stack([cof(1, 1, 2, 2), -cof(0, 1, 2, 2), cof(0, 1, 1, 2)]),
            torch.stack([-cof(1, 0, 2, 2), cof(0, 0, 2, 2), -cof(0, 0, 1, 2)]),
            torch.stack([cof(1, 0, 2, 1), -cof(0, 0, 2, 1), cof(0, 0, 1, 1)]),
        ])
        J = jac[0, 0] * GJ[0, 0] + jac[0, 1] * GJ[1, 0] + jac[0, 2] * GJ[2, 0]
    if check:
        bad = J <= 0
        if bool(bad.any()):
            k, q = [int(v) for v in torch.nonzero(bad)[0]]
            raise NonPositiveJacobian(k + k_offset, q, float(J[k, q]))

    xf = torch.einsum("qn,knd->dkq", mops["Ef"], X)
    jf = torch.einsum("aqn,knd->dakq", mops["Efg"], X)       # (dim, dim, Kc, F)
    Kc, F = jf.shape[2], jf.shape[3]
    nf = mops["tangents"].shape[0]
    nfq = F // nf
    tan = mops["tangents"]                                   # (nf, dim-1, dim)
    jf = jf.reshape(dim, dim, Kc, nf, nfq)
    # physical tangents: T[m, d] = sum_a jac[d, a] * tan[f, m, a]
    T = torch.einsum("dakfq,fma->mdkfq", jf, tan)
    if dim == 2:
        t = T[0]
        sJ = torch.sqrt(t[0] ** 2 + t[1] ** 2)
        n = torch.stack([t[1] / sJ, -t[0] / sJ])
    else:
        a, b = T[0], T[1]
        c = torch.stack([a[1] * b[2] - a[2] * b[1],
                         a[2] * b[0] - a[0] * b[2],
                         a[0] * b[1] - a[1] * b[0]])
        sJ = torch.sqrt(c[0] ** 2 + c[1] ** 2 + c[2] ** 2)
        n = c / sJ
    return {"xq": xq, "J": J, "GJ": GJ, "xf": xf,
            "sJ": sJ.reshape(Kc, F), "n": n.reshape(dim, Kc, F)}


def compute_geometric_data(mesh, ref):
    """Host evaluation of the mapping metric (reference-compatible API,
    R/.../geometry.py:56-102).  Raises NonPositiveJacobian."""
    if mesh.shape.dim == 2:
        return _host_geometry_2d(mesh, ref)
    mops = map_operators(mesh.shape, mesh.N_geo, ref).to("cpu")
    X = torch.as_tensor(np.asarray(mesh.elem_map_nodes, dtype=np.float64))
    g = geometric_factors(X, mops)
    J = g["J"].numpy()
    G = (g["GJ"] / g["J"]).numpy()
    return GeometricData(
        ref=ref, xyzq=tuple(g["xq"].numpy()), Jq=J, Gq=G,
        xyzfq=tuple(g["xf"].numpy()), Jfq=g["sJ"].numpy(), nq=tuple(g["n"].numpy()))


def element_areas(geo):
    return geo.Jq @ geo.ref.wq


def element_perimeters(geo):
    return geo.Jfq @ geo.ref.wfq


def _host_geometry_2d(mesh, ref):
    """2D host metric with per-coordinate BLAS products (the reference's
    matrix formulation, R/.../geometry.py:56-102), so the host diagnostics
    (w_upd_p, geo, stable_dt) agree with the reference to rounding of the same
    operations: J = x_r y_s - x_s y_r, (dr/dx) = [y_s, -x_s; -y_r, x_r] / J,
    face normal (y', -x') / |.| along each face's CCW parameter."""
    mo = map_operators(mesh.shape, mesh.N_geo, ref)
    X = np.asarray(mesh.elem_map_nodes[:, :, 0], dtype=np.float64)
    Y = np.asarray(mesh.elem_map_nodes[:, :, 1], dtype=np.float64)
    Er, Es = mo.Eg
    xq, yq = X @ mo.E.T, Y @ mo.E.T
    xr, xs, yr, ys = X @ Er.T, X @ Es.T, Y @ Er.T, Y @ Es.T
    J = xr * ys - xs * yr
    if np.any(J <= 0):
        k, q = np.argwhere(J <= 0)[0]
        raise NonPositiveJacobian(int(k), int(q), float(J[k, q]))
    G = np.stack([np.stack([ys / J, -xs / J]), np.stack([-yr / J, xr / J])])
    Efr, Efs = mo.Efg
    xf, yf = X @ mo.Ef.T, Y @ mo.Ef.T
    xfr, xfs, yfr, yfs = X @ Efr.T, X @ Efs.T, Y @ Efr.T, Y @ Efs.T
    tx, ty = np.empty_like(xf), np.empty_like(xf)
    nfq = ref.nfq
    for f in range(mesh.shape.n_faces):
        dr, ds = mo.tangents[f][0]
        sl = slice(f * nfq, (f + 1) * nfq)
        tx[:, sl] = xfr[:, sl] * dr + xfs[:, sl] * ds
        ty[:, sl] = yfr[:, sl] * dr + yfs[:, sl] * ds
    sJ = np.hypot(tx, ty)
    return GeometricData(ref=ref, xyzq=(xq, yq), Jq=J, Gq=G, xyzfq=(xf, yf), Jfq=sJ,
                         nq=(ty / sJ, -tx / sJ))
