"""Curved isoparametric meshes: the reference's container and interchange
format, plus the synthetic warped triangle / tetrahedral meshes of
BASELINE.json's configs (the reference ships quadrilateral generators only,
SURVEY.md §0.4).

Container conventions follow R/pkg/src/wadg/meshgen.py:43-67:
``elem_map_nodes`` (K, Npg, dim) physical coordinates of the degree-N_geo
reference node set, ``face_connectivity`` (K, nf, 2) = (neighbour element,
neighbour face) or (-1, -1), ``boundary_tags`` (K, nf) > 0 = Dirichlet.
New here: ``face_orientation`` (K, nf), the code c of
``refelem.orientation_permutations`` relating the two sides of an interior
face (2D conforming CCW meshes always use reversal, code 1, which is the
reference's ``nfq-1-i`` gather, R/.../solver.py:181-193).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import refelem
from .refelem import ElementShape

MESH_SCHEMA_VERSION = "wadg-mesh-v1"
BOUNDARY_NONE = 0
BOUNDARY_DIRICHLET = 1


@dataclass
class CurvedMesh:
    shape: ElementShape
    N_geo: int
    elem_map_nodes: np.ndarray = field(repr=False)
    face_connectivity: np.ndarray = field(repr=False)
    boundary_tags: np.ndarray = field(repr=False)
    h: float = 0.0
    provenance: dict = field(default_factory=dict)
    face_orientation: np.ndarray | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.face_orientation is None:
            # conforming CCW 2D meshes: every interior face is a reversal
            if self.shape.dim != 2:
                raise ValueError("3D meshes need face_orientation")
            self.face_orientation = np.where(self.face_connectivity[:, :, 0] >= 0, 1, 0)

    @property
    def K(self):
        return self.elem_map_nodes.shape[0]

    @property
    def n_faces(self):
        return self.shape.n_faces

    @property
    def dim(self):
        return self.shape.dim


CurvedMesh2D = CurvedMesh   # reference name


def build_connectivity(elem_vertices, shape):
    """Match faces by their (sorted) global vertex ids.

    elem_vertices: (K, n_vertices) int global ids in reference-vertex order.
    Returns (face_connectivity (K, nf, 2), boundary_tags (K, nf),
    face_orientation (K, nf))."""
    elem_vertices = np.asarray(elem_vertices, dtype=np.int64)
    K = elem_vertices.shape[0]
    fv = np.array(refelem.face_vertices(shape))                  # (nf, nvf)
    nf, nvf = fv.shape
    fverts = elem_vertices[:, fv]                                # (K, nf, nvf)
    keys = np.sort(fverts, axis=2).reshape(K * nf, nvf)
    nbits = max(1, int(elem_vertices.max()).bit_length())
    if nbits * nvf <= 62:       # one packed int64 key per face: a single sort instead of a lexsort
        packed = np.zeros(K * nf, dtype=np.int64)
        for c in range(nvf):
            packed = (packed << nbits) | keys[:, c]
        order = np.argsort(packed, kind="stable")
        sp = packed[order]
        same = sp[1:] == sp[:-1]
    else:
        order = np.lexsort(keys.T[::-1])
        sk = keys[order]
        same = np.all(sk[1:] == sk[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("non-manifold mesh: a face is shared by more than two elements")
    conn = np.full((K * nf, 2), -1, dtype=np.int64)
    a = order[:-1][same]
    b = order[1:][same]
    conn[a, 0], conn[a, 1] = b // nf, b % nf
    conn[b, 0], conn[b, 1] = a // nf, a % nf
    conn = conn.reshape(K, nf, 2)
    tags = np.where(conn[:, :, 0] < 0, BOUNDARY_DIRICHLET, BOUNDARY_NONE).astype(np.int64)

    # orientation: pi[n] = m with my face vertex m == neighbour face vertex n
    perms = refelem.orientation_permutations(shape)
    lut = {p: c for c, p in enumerate(perms)}
    orient = np.zeros((K, nf), dtype=np.int64)
    kk, ff = np.nonzero(conn[:, :, 0] >= 0)
    mine = fverts[kk, ff]                                        # (M, nvf)
    nbr = fverts[conn[kk, ff, 0], conn[kk, ff, 1]]
    match = nbr[:, :, None] == mine[:, None, :]                  # [n, m]
    pi = np.argmax(match, axis=2)
    # encode each permutation in base nvf and map through a lookup table
    table = np.full(nvf ** nvf, -1, dtype=np.int64)
    for p, c in lut.items():
        table[sum(v * nvf ** n for n, v in enumerate(p))] = c
    key = (pi * (nvf ** np.arange(nvf))[None, :]).sum(axis=1)
    codes = table[key]
    if np.any(codes < 0):
        raise ValueError("inconsistent face vertex matching")
    orient[kk, ff] = codes
    return conn, tags, orient


def _simplex_map_nodes(shape, N_geo, corner_xyz):
    """Affine placement of the reference node set in each simplex.
    corner_xyz: (K, dim+1, dim) physical vertices in reference-vertex order
    (numpy, or a torch tensor for large meshes: one multi-threaded matmul)."""
    nodes = refelem.interpolation_nodes(shape, N_geo)
    lam_rest = 0.5 * (1.0 + nodes)                                # (Npg, dim)
    lam = np.concatenate([1.0 - lam_rest.sum(axis=1, keepdims=True), lam_rest], axis=1)
    if isinstance(corner_xyz, torch.Tensor):
        return torch.matmul(torch.from_numpy(lam).to(corner_xyz.dtype), corner_xyz)   # (K, Npg, dim)
    return np.einsum("nv,kvd->knd", lam, corner_xyz)


def warp_config1(x, y, amp=0.125):
    """BASELINE config 1 warp (boundary-fixing on [-1, 1]^2)."""
    dx = amp * np.cos(np.pi * x / 2) * np.cos(3 * np.pi * y / 2)
    dy = amp * np.sin(np.pi * x) * np.cos(np.pi * y / 2)
    return x + dx, y + dy


def warped_triangle_mesh(K1D=16, N_geo=4, amp=0.125, domain=((-1.0, 1.0), (-1.0, 1.0))):
    """K1D x K1D squares, each split along its (x0,y0)-(x1,y1) diagonal into
    two CCW triangles, degree-N_geo nodes warped by ``warp_config1``
    (BASELINE config 1: K1D=16, N_geo=N=4, amp=0.125, h = 2/K1D)."""
    (x0, x1), (y0, y1) = domain
    gx = np.linspace(x0, x1, K1D + 1)
    gy = np.linspace(y0, y1, K1D + 1)
    vid = lambda i, j: j * (K1D + 1) + i
    tris = []
    for j in range(K1D):
        for i in range(K1D):
            tris.append((vid(i, j), vid(i + 1, j), vid(i + 1, j + 1)))
            tris.append((vid(i, j), vid(i + 1, j + 1), vid(i, j + 1)))
    tris = np.array(tris, dtype=np.int64)
    VX, VY = np.meshgrid(gx, gy, indexing="xy")
    verts = np.column_stack([VX.ravel(), VY.ravel()])
    X = _simplex_map_nodes(ElementShape.Triangle, N_geo, verts[tris])
    if amp != 0.0:
        wx, wy = warp_config1(X[..., 0], X[..., 1], amp)
        X = np.stack([wx, wy], axis=-1)
    conn, tags, orient = build_connectivity(tris, ElementShape.Triangle)
    h = (x1 - x0) / K1D
    prov = {"kind": "warped-triangle", "K1D": K1D, "N_geo": N_geo, "amp": amp}
    return CurvedMesh(ElementShape.Triangle, N_geo, np.ascontiguousarray(X), conn, tags,
                      h=h, provenance=prov, face_orientation=orient)


def uniform_quad_mesh(K1D, domain=((-1.0, 1.0), (-1.0, 1.0)), N_geo=1):
    """K1D x K1D affine quadrilateral mesh (R/.../meshgen.py:143-154)."""
    (x0, x1), (y0, y1) = domain
    nodes = refelem.quad_nodes(N_geo)
    gx = np.linspace(x0, x1, K1D + 1)
    gy = np.linspace(y0, y1, K1D + 1)
    X = []
    quads = []
    vid = lambda i, j: j * (K1D + 1) + i
    for j in range(K1D):
        for i in range(K1D):
            cx = gx[i] + 0.5 * (nodes[:, 0] + 1) * (gx[i + 1] - gx[i])
            cy = gy[j] + 0.5 * (nodes[:, 1] + 1) * (gy[j + 1] - gy[j])
            X.append(np.column_stack([cx, cy]))
            quads.append((vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)))
    conn, tags, orient = build_connectivity(np.array(quads), ElementShape.Quadrilateral)
    h = float(np.hypot((x1 - x0) / K1D, (y1 - y0) / K1D))
    prov = {"kind": "uniform", "K1D": K1D, "domain": domain, "N_geo": N_geo}
    return CurvedMesh(ElementShape.Quadrilateral, N_geo, np.array(X), conn, tags,
                      h=h, provenance=prov, face_orientation=orient)


# ---------------------------------------------------------------------------
# 3D: Kuhn-split warped cube

# the six Kuhn tetrahedra of a unit cube share the (0,0,0)-(1,1,1) diagonal;
# each walks the cube edges along one permutation of the axes
_KUHN_PATHS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


def _kuhn_local():
    out = []
    for p in _KUHN_PATHS:
        v = [np.zeros(3, dtype=np.int64)]
        for ax in p:
            w = v[-1].copy()
            w[ax] = 1
            v.append(w)
        v = np.array(v)
        if np.linalg.det((v[1:] - v[0]).astype(float)) < 0:
            v[[1, 2]] = v[[2, 1]]
        out.append(v)
    return np.array(out)        # (6, 4, 3) corner offsets, positively oriented


def warp_cube(x, y, z, amp=0.1):
    """BASELINE configs 2-5 warp, read as cyclic permutations:
    x += a cos(pi x/2) cos(3 pi y/2) cos(pi z/2), y and z cyclically.
    Works on numpy arrays or torch tensors; each cosine is evaluated once."""
    cos = torch.cos if isinstance(x, torch.Tensor) else np.cos
    cx, cy, cz = (cos(0.5 * np.pi * v) for v in (x, y, z))
    c3x, c3y, c3z = (cos(1.5 * np.pi * v) for v in (x, y, z))
    return (x + amp * cx * c3y * cz,
            y + amp * cy * c3z * cx,
            z + amp * cz * c3x * cy)


def warped_cube_tet_mesh(n, N_geo, amp=0.1, nz=None, z_range=None, domain=(-1.0, 1.0), z_grid=None):
    """n x n x nz cubes on [-1,1]^2 x z_range, 6 Kuhn tets each, element
    order (kz, tet, ky, kx): z-major so z-slabs are contiguous ranges, and
    within a z-layer grouped by Kuhn tet type, so that consecutive elements
    (one warp of a kernel) are the same tet type in consecutive cubes and
    their neighbours across any local face are consecutive elements with one
    common face code: neighbour-trace gathers are coalesced.

    Default nz = n and z_range = domain (the cube of configs 2-4).  For the
    weak-scaling config 5 pass nz = 48*G and z_range = (-1, -1 + 2*nz/n) ...
    the warp is evaluated in physical coordinates in any case.  ``z_grid``
    (nz + 1 values) gives the layer planes explicitly (a slab of a larger mesh,
    with node coordinates bitwise equal to the larger mesh's)."""
    lo, hi = domain
    hx = (hi - lo) / n
    gx = lo + hx * np.arange(n + 1)
    if z_grid is not None:
        gz = np.asarray(z_grid, dtype=np.float64)
        nz = len(gz) - 1
        zlo, zhi = float(gz[0]), float(gz[-1])
    else:
        nz = n if nz is None else nz
        zlo, zhi = (lo, hi) if z_range is None else z_range
        gz = np.linspace(zlo, zhi, nz + 1)
    local = _kuhn_local()                                           # (6, 4, 3)
    kz, ky, kx = np.meshgrid(np.arange(nz), np.arange(n), np.arange(n), indexing="ij")
    base = np.stack([kx.ravel(), ky.ravel(), kz.ravel()], axis=1)   # (C, 3) z-major
    corners = base[:, None, None, :] + local[None]                  # (C, 6, 4, 3)
    corners = corners.reshape(nz, n * n, 6, 4, 3).transpose(0, 2, 1, 3, 4).reshape(-1, 4, 3)
    vid = (corners[..., 2] * (n + 1) + corners[..., 1]) * (n + 1) + corners[..., 0]
    xyz = np.stack([gx[corners[..., 0]], gx[corners[..., 1]], gz[corners[..., 2]]], axis=-1)
    # torch (multi-threaded) for the node placement and the ~10^8 cosines of a 1.5M-tet mesh
    X = _simplex_map_nodes(ElementShape.Tetrahedron, N_geo, torch.from_numpy(xyz))
    if amp != 0.0:
        X = torch.stack(warp_cube(X[..., 0], X[..., 1], X[..., 2], amp), dim=-1)
    X = X.numpy()
    conn, tags, orient = build_connectivity(vid, ElementShape.Tetrahedron)
    prov = {"kind": "warped-kuhn-cube", "n": n, "nz": nz, "N_geo": N_geo, "amp": amp,
            "z_range": [float(zlo), float(zhi)]}
    return CurvedMesh(ElementShape.Tetrahedron, N_geo, np.ascontiguousarray(X), conn, tags,
                      h=hx, provenance=prov, face_orientation=orient)


def replicate_mesh(mesh, copies):
    """``copies`` disjoint copies of ``mesh`` in one mesh (element k of copy b is
    element b*K + k; neighbours stay within their copy).  Used to evaluate many
    independent right-hand sides in one device pass (analysis.assemble_evolution_matrix)."""
    K = mesh.K
    off = (np.arange(copies, dtype=np.int64) * K)[:, None, None]
    conn = np.broadcast_to(mesh.face_connectivity[None], (copies,) + mesh.face_connectivity.shape).copy()
    inner = conn[..., 0] >= 0
    conn[..., 0] = np.where(inner, conn[..., 0] + off, -1)
    rep = lambda a: np.ascontiguousarray(np.broadcast_to(a[None], (copies,) + a.shape).reshape((copies * K,) + a.shape[1:]))
    return CurvedMesh(mesh.shape, mesh.N_geo, rep(mesh.elem_map_nodes), conn.reshape(copies * K, -1, 2),
                      rep(mesh.boundary_tags), h=mesh.h, provenance=dict(mesh.provenance, copies=copies),
                      face_orientation=rep(np.asarray(mesh.face_orientation)))


# ---------------------------------------------------------------------------
# Interchange (R/.../meshgen.py:485-517, extended with shape "tetrahedron"
# and the face_orientation array)

def save_mesh(mesh, path):
    doc = {
        "version": MESH_SCHEMA_VERSION, "shape": mesh.shape.value, "N_geo": mesh.N_geo,
        "K": mesh.K, "h": mesh.h, "elem_map_nodes": mesh.elem_map_nodes.tolist(),
        "face_connectivity": mesh.face_connectivity.tolist(),
        "boundary_tags": mesh.boundary_tags.tolist(),
        "face_orientation": np.asarray(mesh.face_orientation).tolist(),
        "provenance": mesh.provenance,
    }
    with open(path, "w") as f:
        json.dump(doc, f)


def load_mesh(path):
    with open(path) as f:
        doc = json.load(f)
    if doc.get("version") != MESH_SCHEMA_VERSION:
        raise ValueError(f"unsupported mesh schema version {doc.get('version')!r}")
    shape = ElementShape(doc["shape"])
    nodes = np.asarray(doc["elem_map_nodes"], dtype=float)
    conn = np.asarray(doc["face_connectivity"], dtype=np.int64)
    tags = np.asarray(doc["boundary_tags"], dtype=np.int64)
    npg = refelem.basis_dimension(shape, doc["N_geo"])
    if nodes.shape != (doc["K"], npg, shape.dim):
        raise ValueError("elem_map_nodes shape inconsistent with K and N_geo")
    if conn.shape != (doc["K"], shape.n_faces, 2) or tags.shape != (doc["K"], shape.n_faces):
        raise ValueError("connectivity arrays inconsistent with K")
    orient = doc.get("face_orientation")
    orient = None if orient is None else np.asarray(orient, dtype=np.int64)
    return CurvedMesh(shape=shape, N_geo=doc["N_geo"], elem_map_nodes=nodes,
                      face_connectivity=conn, boundary_tags=tags, h=float(doc["h"]),
                      provenance=doc.get("provenance", {}), face_orientation=orient)
