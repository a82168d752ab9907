"""Device-resident problem data: packs reference operators and per-element
geometry into the HBM layout the kernels expect and fills the
``wadg_problem`` C struct (include/wadg_b200.h).

Layout (element index fastest, padded to Kpad, a multiple of 128):

* fields        Q, res, rhs    (dim+1, Np, Kpad)
* volume geo    (dr_a/dx_i) J  (dim*dim, Nq, Kpad)
* face geo      n_i, sJ/2      (dim+1, Nf*Nfq, Kpad)
* update wts    1/J, c^2/J     (Nqu, Kpad) each (c^2/J only for a variable c^2)
* neighbours    nbr, ncode     (Nf, Kpad) int32

Per-element geometry is computed on the target device in element chunks
straight from the map nodes, so million-element meshes never materialise
(K, Nq) float64 arrays on the host (SURVEY.md §7 hard part 5).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native, geometry, refelem
from .errors import ConfigError

PAD = 384        # element padding: a multiple of every fused block size (128, 64, 32, 24, 16)
CHUNK = 1 << 16


def roundup(n, m):
    return ((n + m - 1) // m) * m


def torch_dtype(name):
    return {"float64": torch.float64, "float32": torch.float32}[str(name)]


class HaloPlan:
    """Halo description for an element range of a partitioned mesh.

    recv_slot: dict (local k, f) -> halo slot; send_k/send_f: int32 arrays of
    the faces this rank packs (in message order); peers: list of
    (rank, n_send, n_recv) in message order."""

    def __init__(self, recv_slot, send_k, send_f, peers):
        self.recv_slot = recv_slot
        self.send_k = np.asarray(send_k, dtype=np.int32)
        self.send_f = np.asarray(send_f, dtype=np.int32)
        self.peers = peers

    @property
    def n_recv(self):
        return len(self.recv_slot)


def neighbour_tables(mesh, n_orient, k0=0, k1=None, halo=None):
    """nbr / ncode (Nf, K_local) for elements [k0, k1) of ``mesh``."""
    k1 = mesh.K if k1 is None else k1
    conn = mesh.face_connectivity[k0:k1]
    orient = mesh.face_orientation[k0:k1]
    kk = conn[:, :, 0]
    nbr = np.where(kk >= 0, kk - k0, -1).astype(np.int64)
    ncode = np.where(kk >= 0, conn[:, :, 1] * n_orient + orient, 0).astype(np.int64)
    outside = (kk >= 0) & ((kk < k0) | (kk >= k1))
    if np.any(outside):
        if halo is None:
            raise ValueError("element range has off-range neighbours but no halo plan")
        for k, f in zip(*np.nonzero(outside)):
            nbr[k, f] = -2 - halo.recv_slot[(int(k), int(f))]
    return nbr.T.astype(np.int32), ncode.T.astype(np.int32)


def interleave_blocks(x, npad, blk=128):
    """(rows, npts, Kpad) element-fastest -> (Kpad/blk, rows, npad/4, blk, 4):
    per 128-element block, 4 consecutive points of one element are 16
    contiguous bytes and a warp's 32 elements read 512 contiguous bytes
    (include/wadg_b200.h, *_il).  Points npts..npad are zero."""
    rows, npts, Kp = x.shape
    xp = torch.zeros((rows, npad, Kp), dtype=x.dtype, device=x.device)
    xp[:, :npts] = x
    out = xp.view(rows, npad // 4, 4, Kp // blk, blk).permute(3, 0, 1, 4, 2).contiguous()
    del xp
    return out


def medium_on_device(c2, xq, shape):
    """c^2 at the points xq (torch tensors on the device), as a float64 tensor
    of ``shape``.  A callable is evaluated on the device tensors (torch
    expressions stay on the GPU); a numpy-only callable falls back to a host
    evaluation of the same points.  Non-positive or non-finite values raise
    ConfigError, like the reference's MediumField (R/.../solver.py:62-63)."""
    dev = xq[0].device
    if not callable(c2):
        v = torch.full(shape, float(c2), dtype=torch.float64, device=dev)
    else:
        try:
            v = c2(*xq)
            if not isinstance(v, torch.Tensor):
                raise TypeError("numpy result")
            v = v.to(device=dev, dtype=torch.float64).expand(shape)
        except (TypeError, RuntimeError, AttributeError):
            xyz = [a.cpu().numpy() for a in xq]
            v = torch.as_tensor(np.array(np.broadcast_to(np.asarray(c2(*xyz), dtype=float), shape)), device=dev)
    if not bool(torch.all(torch.isfinite(v) & (v > 0))):
        raise ConfigError("wavespeed squared must be positive")
    return v


def tf32_split(a, mode=None):
    """fp32 x = hi + lo exactly, hi a tf32 value: x rounded to the nearest
    tf32 (ties away, "rn", default) or with the low 13 mantissa bits cleared
    ("trunc", the tensor core's own view of a raw fp32 operand)."""
    mode = mode or os.environ.get("WADG_TF32_SPLIT", "rn")
    x = np.ascontiguousarray(a, dtype=np.float32)
    bits = x.view(np.uint32)
    if mode == "rn":
        bits = bits + np.uint32(0x1000)
    hi = (bits & np.uint32(0xFFFFE000)).view(np.float32)
    return hi, (x - hi).astype(np.float32)


def kmajor_image(B):
    """Canonical K-major no-swizzle UMMA image of B (rows x K), rows % 8 == 0,
    K % 4 == 0: 8-row x 4-value core matrices of 128 contiguous bytes, core
    matrices adjacent along K contiguous (LBO = 128 B), 8-row groups
    (K/4)*128 B apart (csrc/wadg_umma.cuh)."""
    R, KT = B.shape
    assert R % 8 == 0 and KT % 4 == 0
    return B.reshape(R // 8, 8, KT // 4, 4).transpose(0, 2, 1, 3).ravel()


def split_images(*blocks):
    """hi images of all blocks, then lo images (one operator tile)."""
    his, los = zip(*(tf32_split(b) for b in blocks))
    return np.concatenate([kmajor_image(h) for h in his] + [kmajor_image(lo) for lo in los])


def umma_operator_images(ref, ru, cfg):
    """All reference operators of the tcgen05 fused stage (csrc/wadg_fused_umma.cuh,
    CfgU offsets): per volume chunk D_a, DTW_a, -Pq and per chunk pair Vq; Vfi per
    16-point half of the face rule; -Pf per face and half; update chunks Vu, Pu."""
    NP, NQ = ref.Np, ref.Nq
    QC, NCH, NPK, NPN, NFPK, NFH = cfg["qc"], cfg["nch"], cfg["npp"], cfg["qcs"], cfg["njs"], cfg["nfq8"]
    QU = 16
    NCHU = -(-NQ // QU)
    nf, nfq, nfp = ref.n_faces, ref.nfq, ref.nfp
    DTW = [ref.Mhat_inv @ D.T @ np.diag(ref.wq) for D in ref.Dq]

    def rows(M, r0, n, kt):                 # rows r0.. r0+n of M (zero past the end), K padded to kt
        out = np.zeros((n, kt))
        r1 = min(M.shape[0], r0 + n)
        if r1 > r0:
            out[:r1 - r0, :M.shape[1]] = M[r0:r1]
        return out

    parts = []
    for ch in range(NCH):                   # D_a: rows a*16 + qq
        parts.append(split_images(np.vstack([rows(D, ch * QC, QC, NPK) for D in ref.Dq])))
    for pr in range(-(-NCH // 2)):          # Vq: rows qq of a chunk pair (2 QC quadrature points)
        parts.append(split_images(rows(ref.Vq, pr * 2 * QC, 2 * QC, NPK)))
    for ch in range(NCH):                   # DTW_a: 3 blocks of (NPN rows j) x (QC columns q)
        parts.append(split_images(*[rows(M.T, ch * QC, QC, NPN).T for M in DTW]))
    for ch in range(NCH):                   # -Pq: (NPN rows j) x (QC columns q)
        parts.append(split_images(rows(-ref.Pq.T, ch * QC, QC, NPN).T))
    for hh in range(NFH):                   # Vfi per 16-point half of the face rule
        parts.append(split_images(rows(ref.face_interp, hh * 16, 16, NFPK)))
    for f in range(nf):                     # -Pf per face and half
        for hh in range(NFH):
            parts.append(split_images(rows((-ref.Pfq[:, f * nfq:(f + 1) * nfq]).T, hh * 16, 16, NPN).T))
    for u in range(NCHU):
        parts.append(split_images(rows(ru.Vq, u * QU, QU, NPK)))
    for u in range(NCHU):
        parts.append(split_images(rows(ru.Pq.T, u * QU, QU, NPN).T))
    out = np.concatenate(parts).astype(np.float32)
    assert nfp <= NFPK
    return out


def frag_image(B, K, Nn):
    """DMMA (mma.m8n8k4.f64) B-fragment image of B (k x n, zero padded to
    K x Nn): [K/4][Nn/8][32], lane t holding B[4 ks + t % 4][8 nt + t // 4]
    (csrc/wadg_fused_dmma.cuh)."""
    Bp = np.zeros((K, Nn))
    Bp[:B.shape[0], :B.shape[1]] = B
    lane = np.arange(32)
    ks, nt = np.arange(K // 4), np.arange(Nn // 8)
    kk = 4 * ks[:, None, None] + (lane % 4)[None, None, :]
    nn = 8 * nt[None, :, None] + (lane // 4)[None, None, :]
    return Bp[kk, nn]


def reg_operator_image(ref, ru, DTW, total):
    """The reference-operator values of the thread-per-element register stage
    (csrc/wadg_fused_reg.cuh, rk::CfgR offsets; 464 at N = 1): D_a [a][q][j],
    Vq [q][j], DTW_a^T [q][a][j], Pq^T [q][j], the own-trace interpolation Vfi
    applied to the face nodes [f][fq][j], Vfi [fq][i], Pf^T [f][fq][j], and the
    update rule's Vu [q][j] and Pu^T [q][j]; node rows padded to rup(Np, 4),
    face-node rows to rup(Nfp, 4), with zeros."""
    nf, nfq, Np, nfp = ref.n_faces, ref.nfq, ref.Np, ref.nfp
    NPS, NFPS = roundup(Np, 4), roundup(nfp, 4)

    def rows(a, width):           # pad the last axis to `width`
        a = np.asarray(a, dtype=np.float64)
        out = np.zeros(a.shape[:-1] + (width,))
        out[..., :a.shape[-1]] = a
        return out
    Vfi = np.asarray(ref.face_interp)
    VF = np.zeros((nf, nfq, Np))
    for f in range(nf):
        VF[f][:, list(ref.face_nodes[f])] = Vfi
    parts = [rows(np.stack(list(ref.Dq)), NPS), rows(ref.Vq, NPS), rows(np.stack(DTW, axis=0).transpose(2, 0, 1), NPS),
             rows(ref.Pq.T, NPS), rows(VF, NPS), rows(Vfi, NFPS), rows(np.asarray(ref.Pfq).T.reshape(nf, nfq, Np), NPS),
             rows(ru.Vq, NPS), rows(ru.Pq.T, NPS)]
    img = np.concatenate([np.ascontiguousarray(x).ravel() for x in parts])
    assert img.size == total, (img.size, total)
    return img


def dmma_operator_images(ref, ru, cfg, strong_weak=True):
    """All reference operators of the DMMA fused stage (csrc/wadg_fused_dmma.cuh,
    CfgD offsets), in fragment order: per volume chunk D_r, D_s, D_t (, Vq) (k =
    node, n = point) and (DTW_r, DTW_s, DTW_t,) -Pq (k = point, n = node); Vfi;
    -Pf per face; per update chunk Vu and Pu.  The strong form has no Vq / DTW
    images (its volume term is -Pq sum_i sum_a G_ai D_a u_i)."""
    NP, NQ = ref.Np, ref.Nq
    QC, NCH, NPP, NFPK, NFQP = cfg["qc"], cfg["nch"], cfg["npp"], cfg["qcs"], cfg["njs"]
    NCHU = -(-ru.Nq // QC)
    nf, nfq = ref.n_faces, ref.nfq
    DTW = [ref.Mhat_inv @ D.T @ np.diag(ref.wq) for D in ref.Dq]
    va = list(ref.Dq) + ([ref.Vq] if strong_weak else [])
    vb = (DTW if strong_weak else []) + [-ref.Pq]

    def cols(M, c0, n):                     # columns c0 .. c0+n of M (zero past the end)
        out = np.zeros((M.shape[0], n))
        c1 = min(M.shape[1], c0 + n)
        if c1 > c0:
            out[:, :c1 - c0] = M[:, c0:c1]
        return out

    parts = []
    for ch in range(NCH):
        parts += [frag_image(cols(Op.T, ch * QC, QC), NPP, QC) for Op in va]
    for ch in range(NCH):
        parts += [frag_image(cols(Op, ch * QC, QC).T, QC, NPP) for Op in vb]
    parts.append(frag_image(ref.face_interp.T, NFPK, NFQP))
    for f in range(nf):
        parts.append(frag_image(-ref.Pfq[:, f * nfq:(f + 1) * nfq].T, NFQP, NPP))
    for ch in range(NCHU):
        parts.append(frag_image(cols(ru.Vq.T, ch * QC, QC), NPP, QC))
    for ch in range(NCHU):
        parts.append(frag_image(cols(ru.Pq, ch * QC, QC).T, QC, NPP))
    out = np.concatenate([p.ravel() for p in parts])
    assert out.size == cfg["nfq8"], (out.size, cfg["nfq8"])
    return out


def tmma_frag_image(B, K, Nn):
    """split-TF32 mma.sync m16n8k8 B-fragment image of B (k x n, zero padded to
    K x Nn): [K/8][Nn/8][32][4], lane (g = lane // 4, t = lane % 4) holding
    hi(B[8ks+t][8nt+g]), hi(B[8ks+t+4][8nt+g]) and the two lo parts, hi / lo
    the round-to-nearest tf32 split (csrc/wadg_fused_tmma.cuh)."""
    Bp = np.zeros((K, Nn))
    Bp[:B.shape[0], :B.shape[1]] = B
    lane = np.arange(32)
    ks, nt = np.arange(K // 8), np.arange(Nn // 8)
    kk = 8 * ks[:, None, None] + (lane % 4)[None, None, :]
    nn = 8 * nt[None, :, None] + (lane // 4)[None, None, :]
    hi, lo = tf32_split(Bp, "rn")
    return np.stack([hi[kk, nn], hi[kk + 4, nn], lo[kk, nn], lo[kk + 4, nn]], axis=-1)


def tmma_operator_images(ref, ru, cfg, strong_weak=True):
    """All reference operators of the split-TF32 mma.sync stage (CfgT offsets),
    in the order of dmma_operator_images (no Vq / DTW images for the strong
    form)."""
    QC, NCH, NPP, NFPK, NFQP = cfg["qc"], cfg["nch"], cfg["npp"], cfg["qcs"], cfg["njs"]
    NCHU = -(-ru.Nq // QC)
    nf, nfq = ref.n_faces, ref.nfq
    DTW = [ref.Mhat_inv @ D.T @ np.diag(ref.wq) for D in ref.Dq]
    va = list(ref.Dq) + ([ref.Vq] if strong_weak else [])
    vb = (DTW if strong_weak else []) + [-ref.Pq]

    def cols(M, c0, n):
        out = np.zeros((M.shape[0], n))
        c1 = min(M.shape[1], c0 + n)
        if c1 > c0:
            out[:, :c1 - c0] = M[:, c0:c1]
        return out

    parts = []
    for ch in range(NCH):
        parts += [tmma_frag_image(cols(Op.T, ch * QC, QC), NPP, QC) for Op in va]
    for ch in range(NCH):
        parts += [tmma_frag_image(cols(Op, ch * QC, QC).T, QC, NPP) for Op in vb]
    parts.append(tmma_frag_image(ref.face_interp.T, NFPK, NFQP))
    for f in range(nf):
        parts.append(tmma_frag_image(-ref.Pfq[:, f * nfq:(f + 1) * nfq].T, NFQP, NPP))
    for ch in range(NCHU):
        parts.append(tmma_frag_image(cols(ru.Vq.T, ch * QC, QC), NPP, QC))
    for ch in range(NCHU):
        parts.append(tmma_frag_image(cols(ru.Pq, ch * QC, QC).T, QC, NPP))
    out = np.concatenate([p.ravel() for p in parts]).astype(np.float32)
    assert out.size == cfg["nfq8"], (out.size, cfg["nfq8"])
    return out


class DeviceProblem:
    """All device arrays of one (mesh range, reference elements, medium) and
    the C struct pointing at them."""

    def __init__(self, mesh, ref, ref_upd, c2, formulation_sw, dtype="float64", device="cuda",
                 k0=0, k1=None, halo=None, exact_mass=False):
        if not torch.cuda.is_available() and str(device).startswith("cuda"):
            raise RuntimeError("paper_1608_03836_b200 needs a CUDA device (no CPU fallback)")
        _native.load()
        self.device = torch.device(device)
        self.dtype = torch_dtype(dtype)
        self.mesh, self.ref, self.ref_upd = mesh, ref, ref_upd
        self.k0 = k0
        self.k1 = mesh.K if k1 is None else k1
        K = self.k1 - self.k0
        self.K, self.Kpad = K, roundup(max(K, 1), PAD)
        self.dim = mesh.shape.dim
        self.fld = self.dim + 1
        self.n_orient = len(refelem.orientation_permutations(mesh.shape))
        self.sw = bool(formulation_sw)
        self.halo = halo
        self._keep = {}
        self._ops()
        self._elements(c2)
        self.halo_buf = None
        if halo is not None and halo.n_recv:
            self.halo_buf = torch.zeros((halo.n_recv, self.fld, ref.nfp), dtype=self.dtype,
                                        device=self.device)
        self.exact_mass = bool(exact_mass)
        self.minv_p = self.minv_u = None
        if self.exact_mass:
            self._exact_mass_operators(c2)
        self.struct = self._make_struct()
        self.fused = None if self.exact_mass else self._fused_ops()
        self._energy_ready = False
        self.energy_partials = torch.empty(self.Kpad // _native.ELEMS_PER_BLOCK, dtype=torch.float64,
                                           device=self.device)
        self.energy_out = torch.empty(1, dtype=torch.float64, device=self.device)

    # -- operators -----------------------------------------------------------
    def _t(self, a, dtype=None):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype or self.dtype,
                               device=self.device)

    def _ops(self):
        ref, ru = self.ref, self.ref_upd
        DTW = np.stack([ref.Mhat_inv @ D.T @ np.diag(ref.wq) for D in ref.Dq])
        fmask = np.array(ref.face_nodes, dtype=np.int64)
        ext = np.empty((ref.n_faces * self.n_orient, ref.nfp), dtype=np.int64)
        for f2 in range(ref.n_faces):
            for o in range(self.n_orient):
                ext[f2 * self.n_orient + o] = fmask[f2][ref.face_perms[o]]
        self.ops = {
            "Vq": self._t(ref.Vq), "Dq": self._t(np.stack(ref.Dq)), "Pq": self._t(ref.Pq),
            "DTW": self._t(DTW), "Vu": self._t(ru.Vq), "Pu": self._t(ru.Pq),
            "Vfi": self._t(ref.face_interp), "Pf": self._t(ref.Pfq),
            "fmask": self._t(fmask, torch.int32), "ext_node": self._t(ext, torch.int32),
            "fperm": self._t(ref.face_perms, torch.int32),
        }

    # -- per-element data ----------------------------------------------------
    def _elements(self, c2):
        ref, ru, dev, dt = self.ref, self.ref_upd, self.device, self.dtype
        dim, K, Kp = self.dim, self.K, self.Kpad
        Nq, F, Nqu = ref.Nq, ref.n_faces * ref.nfq, ru.Nq
        self.geo = torch.zeros((dim * dim, Nq, Kp), dtype=dt, device=dev)
        self.fgeo = torch.zeros((dim + 1, F, Kp), dtype=dt, device=dev)
        self.wu = torch.ones((Nqu, Kp), dtype=dt, device=dev)
        self.variable_c2 = callable(c2)
        self.c2 = 1.0 if self.variable_c2 else float(c2)
        self.wp = torch.ones((Nqu, Kp), dtype=dt, device=dev) if self.variable_c2 else None
        mv = geometry.map_operators(self.mesh.shape, self.mesh.N_geo, ref).to(dev)
        mu = geometry.map_operators(self.mesh.shape, self.mesh.N_geo, ru).to(dev)
        X_all = self.mesh.elem_map_nodes
        for c0 in range(0, K, CHUNK):
            c1 = min(K, c0 + CHUNK)
            X = torch.as_tensor(np.asarray(X_all[self.k0 + c0:self.k0 + c1], dtype=np.float64),
                                device=dev)
            g = geometry.geometric_factors(X, mv, k_offset=self.k0 + c0)
            self.geo[:, :, c0:c1] = g["GJ"].reshape(dim * dim, c1 - c0, Nq).transpose(1, 2).to(dt)
            for i in range(dim):
                self.fgeo[i, :, c0:c1] = g["n"][i].T.to(dt)
            self.fgeo[dim, :, c0:c1] = (0.5 * g["sJ"]).T.to(dt)
            gu = geometry.geometric_factors(X, mu, k_offset=self.k0 + c0)
            Ju = gu["J"]
            self.wu[:, c0:c1] = (1.0 / Ju).T.to(dt)
            if self.variable_c2:
                self.wp[:, c0:c1] = (medium_on_device(c2, gu["xq"], Ju.shape) / Ju).T.to(dt)
            del g, gu, X
        nbr, ncode = neighbour_tables(self.mesh, self.n_orient, self.k0, self.k1, self.halo)
        self.nbr = torch.full((ref.n_faces, Kp), -1, dtype=torch.int32, device=dev)
        self.ncode = torch.zeros((ref.n_faces, Kp), dtype=torch.int32, device=dev)
        self.nbr[:, :K] = torch.as_tensor(nbr, device=dev)
        self.ncode[:, :K] = torch.as_tensor(ncode, device=dev)
        if self.halo is not None and len(self.halo.send_k):
            self.send_k = torch.as_tensor(self.halo.send_k, device=dev)
            self.send_f = torch.as_tensor(self.halo.send_f, device=dev)
            self.send_buf = torch.zeros((len(self.halo.send_k), self.fld, ref.nfp), dtype=dt,
                                        device=dev)

    def _exact_mass_operators(self, c2):
        """ExactCurvedMass comparator (R/.../solver.py:156-167, 302-306): per
        element A = M^-1 Mhat for the J/c^2- (pressure) and J-weighted (velocity)
        mass matrices at quadrature degree 2N + 2 N_geo, assembled, inverted and
        stored on the device in element chunks: (Np, Np, Kpad) each."""
        ref, mesh, dev = self.ref, self.mesh, self.device
        N, Np, K = ref.N, ref.Np, self.K
        ref_m = refelem.build_reference_element(N, mesh.shape, 2 * N + 2 * mesh.N_geo, 1)
        mm = geometry.map_operators(mesh.shape, mesh.N_geo, ref_m).to(dev)
        Vq = torch.as_tensor(ref_m.Vq, dtype=torch.float64, device=dev)
        wq = torch.as_tensor(ref_m.wq, dtype=torch.float64, device=dev)
        Mhat = torch.as_tensor(ref.Mhat, dtype=torch.float64, device=dev)
        self.minv_p = torch.zeros((Np, Np, self.Kpad), dtype=self.dtype, device=dev)
        self.minv_u = torch.zeros((Np, Np, self.Kpad), dtype=self.dtype, device=dev)
        chunk = max(1, min(CHUNK, (1 << 28) // (8 * Np * Np * 4)))
        for c0 in range(0, K, chunk):
            c1 = min(K, c0 + chunk)
            X = torch.as_tensor(np.asarray(self.mesh.elem_map_nodes[self.k0 + c0:self.k0 + c1],
                                           dtype=np.float64), device=dev)
            g = geometry.geometric_factors(X, mm, k_offset=self.k0 + c0)
            J = g["J"]
            cv = medium_on_device(c2, g["xq"], J.shape)
            for w, dst in ((J / cv, self.minv_p), (J, self.minv_u)):
                M = torch.einsum("kq,qi,qj->kij", w * wq, Vq, Vq)
                M = 0.5 * (M + M.transpose(1, 2))
                A = torch.linalg.solve(M, Mhat.expand(M.shape[0], Np, Np))
                dst[:, :, c0:c1] = A.permute(1, 2, 0).to(self.dtype)
            del g, X

    def host_mass_inverses(self):
        """(K, Np, Np) numpy M_k^-1 for pressure and velocity (the reference's
        disc.mass_inv_p / mass_inv_u), recovered from the stored A = M^-1 Mhat."""
        Mi = np.asarray(self.ref.Mhat_inv)
        out = []
        for A in (self.minv_p, self.minv_u):
            a = A[:, :, :self.K].permute(2, 0, 1).to(torch.float64).cpu().numpy()
            out.append(a @ Mi)
        return out

    def _fused_ops(self):
        """Repack the operators for wadg_stage_fused (3D strong-weak with the
        default (N+1)^3 volume/update rules); returns the fused block size or
        None when the fused stage does not apply."""
        ref, ru = self.ref, self.ref_upd
        N = ref.N
        if self.dim != 3 or ru.Nq != (N + 1) ** 3:
            return None
        if self.sw and not (ref.Nq == (N + 1) ** 3 and ref.nfq == (N + 1) ** 2):
            return None
        # strong form: the sufficiency rules at N_geo = N, (2N-1)^3 volume and (2N)^2 face points
        # (the volume rule floored at degree 2N: 2^3 points at N = 1)
        if not self.sw and not (ref.Nq == max(2, 2 * N - 1 if N > 1 else 2) ** 3 and ref.nfq == (2 * N) ** 2):
            return None
        code = _native.WADG_F64 if self.dtype == torch.float64 else _native.WADG_F32
        form = _native.WADG_STRONG_WEAK if self.sw else _native.WADG_STRONG
        cfg = _native.fused_config(code, N, form)
        if cfg is None:
            return None
        kb, qc, nch = cfg["kb"], cfg["qc"], cfg["nch"]
        NP, NQ = ref.Np, ref.Nq
        nf, nfq = ref.n_faces, ref.nfq
        DTW = [ref.Mhat_inv @ D.T @ np.diag(ref.wq) for D in ref.Dq]
        if cfg["kind"] == 2:                    # tcgen05 kernel: one buffer of K-major tile images
            if self.Kpad % kb:
                return None
            packed = umma_operator_images(ref, ru, cfg)
            self.ops["umma"] = self._t(packed, torch.float32)
            for name in ("opVA", "opVB", "opU1", "opU2", "liftT"):
                setattr(self.struct, name, self.ops["umma"].data_ptr())
            # block-interleaved per-element data (include/wadg_b200.h, *_il)
            nch, nchu, nfh = cfg["nch"], -(-ru.Nq // 16), cfg["nfq8"]
            self.geo_il = interleave_blocks(self.geo, nch * 16, kb)
            fg = self.fgeo.view(self.dim + 1, ref.n_faces, ref.nfq, self.Kpad)
            self.fgeo_il = interleave_blocks(fg.reshape((self.dim + 1) * ref.n_faces, ref.nfq, self.Kpad),
                                             nfh * 16, kb)
            # update weights as per-element means wbar plus deviations (wbar in
            # [2][Kpad], include/wadg_b200.h); WADG_WBAR=0 keeps the full weights
            wu, wp = self.wu, self.wp
            self.wbar = None
            if os.environ.get("WADG_WBAR", "1") != "0":
                nq = ru.Nq
                wbu = self.wu[:nq].double().mean(0)
                wbp = self.wp[:nq].double().mean(0) if self.wp is not None else self.c2 * wbu
                self.wbar = torch.stack([wbu, wbp]).to(self.dtype).contiguous()
                wu = self.wu - self.wbar[0]
                wp = self.wp - self.wbar[1] if self.wp is not None else None
            self.wu_il = interleave_blocks(wu.unsqueeze(0), nchu * 16, kb)
            self.wp_il = interleave_blocks(wp.unsqueeze(0), nchu * 16, kb) if wp is not None else None
            del wu, wp
            s = self.struct
            s.geo_il, s.fgeo_il, s.wu_il = self.geo_il.data_ptr(), self.fgeo_il.data_ptr(), self.wu_il.data_ptr()
            s.wp_il = self.wp_il.data_ptr() if self.wp_il is not None else None
            s.wbar = self.wbar.data_ptr() if self.wbar is not None else None
            self.fused_kind = 2
            self.struct.order = N
            self.struct.fused_kind = 2
            return kb
        if cfg["kind"] == 3:                    # DMMA kernel: one buffer of fragment-order images
            if self.Kpad % kb:
                return None
            self.ops["dmma"] = self._t(dmma_operator_images(ref, ru, cfg, self.sw), torch.float64)
            for name in ("opVA", "opVB", "opU1", "opU2", "liftT"):
                setattr(self.struct, name, self.ops["dmma"].data_ptr())
            self.fused_kind = 3
            self.struct.order = N
            self.struct.fused_kind = 3
            return kb
        if cfg["kind"] == 4:                    # split-TF32 mma.sync kernel: fragment-order hi / lo images
            if self.Kpad % kb:
                return None
            self.ops["tmma"] = self._t(tmma_operator_images(ref, ru, cfg, self.sw), torch.float32)
            for name in ("opVA", "opVB", "opU1", "opU2", "liftT"):
                setattr(self.struct, name, self.ops["tmma"].data_ptr())
            self.fused_kind = 4
            self.struct.order = N
            self.struct.fused_kind = 4
            return kb
        if cfg["kind"] == 5:                    # N = 1 thread-per-element kernel: one operator image
            if self.Kpad % kb:
                return None
            self.ops["reg"] = self._t(reg_operator_image(ref, ru, DTW, cfg["nfq8"]))
            for name in ("opVA", "opVB", "opU1", "opU2", "liftT"):
                setattr(self.struct, name, self.ops["reg"].data_ptr())
            self.fused_kind = 5
            self.struct.order = N
            self.struct.fused_kind = 5
            return kb
        # CUDA-core kernel layouts (kind 0)
        NPP = roundup(NP, 4)
        NQP = nch * qc
        A = np.zeros((NQP, NPP, 4))
        A[:NQ, :NP] = np.stack(list(ref.Dq) + [ref.Vq], axis=-1)
        opVA = A.reshape(nch, qc, NPP, 4).transpose(0, 2, 1, 3)
        B = np.zeros((NPP, NQP, 4))
        B[:NP, :NQ] = np.stack(DTW + [ref.Pq], axis=-1)
        opVB = B.reshape(NPP, nch, qc, 4).transpose(1, 2, 0, 3)
        U1 = np.zeros((NQP, NPP))
        U1[:NQ, :NP] = ru.Vq
        opU1 = U1.reshape(nch, qc, NPP).transpose(0, 2, 1)
        U2 = np.zeros((NPP, NQP))
        U2[:NP, :NQ] = ru.Pq
        opU2 = U2.reshape(NPP, nch, qc).transpose(1, 2, 0)
        L = np.zeros((nf * nfq, NPP))
        L[:, :NP] = ref.Pfq.T
        for name, arr in (("opVA", opVA), ("opVB", opVB), ("opU1", opU1), ("opU2", opU2), ("liftT", L)):
            self.ops[name] = self._t(arr)
            setattr(self.struct, name, self.ops[name].data_ptr())
        self.fused_kind = 0
        self.struct.order = N
        self.struct.fused_kind = 0
        if self.Kpad % kb:
            return None
        return kb

    def prepare_energy(self, c2):
        """Energy weights w J / c^2 and w J at the volume rule (diagnostics)."""
        if self._energy_ready:
            return
        ref, dev, dt = self.ref, self.device, self.dtype
        K, Kp, Nq = self.K, self.Kpad, ref.Nq
        self.ewp = torch.zeros((Nq, Kp), dtype=dt, device=dev)
        self.ewu = torch.zeros((Nq, Kp), dtype=dt, device=dev)
        mv = geometry.map_operators(self.mesh.shape, self.mesh.N_geo, ref).to(dev)
        for c0 in range(0, K, CHUNK):
            c1 = min(K, c0 + CHUNK)
            X = torch.as_tensor(np.asarray(self.mesh.elem_map_nodes[self.k0 + c0:self.k0 + c1],
                                           dtype=np.float64), device=dev)
            g = geometry.geometric_factors(X, mv, check=False)
            J = g["J"]
            cv = medium_on_device(c2, g["xq"], J.shape)
            self.ewp[:, c0:c1] = (J / cv).T.to(dt)
            self.ewu[:, c0:c1] = J.T.to(dt)
        self.ops["Ve"] = self._t(ref.Vq)
        self.ops["we"] = self._t(ref.wq)
        s = self.struct
        s.Ne = ref.Nq
        s.Ve, s.we = self.ops["Ve"].data_ptr(), self.ops["we"].data_ptr()
        s.ewp, s.ewu, s.e_recip = self.ewp.data_ptr(), self.ewu.data_ptr(), 0
        self._energy_ready = True

    # -- C struct ------------------------------------------------------------
    def _make_struct(self):
        ref, o = self.ref, self.ops
        s = _native.WadgProblem()
        s.dim, s.dtype = self.dim, (_native.WADG_F64 if self.dtype == torch.float64 else _native.WADG_F32)
        s.K, s.Kpad = self.K, self.Kpad
        s.Np, s.Nq, s.Nqu = ref.Np, ref.Nq, self.ref_upd.Nq
        s.Nf, s.Nfp, s.Nfq = ref.n_faces, ref.nfp, ref.nfq
        s.n_orient = self.n_orient
        s.formulation = _native.WADG_STRONG_WEAK if self.sw else _native.WADG_STRONG
        for name in ("Vq", "Dq", "Pq", "DTW", "Vu", "Pu", "Vfi", "Pf", "fmask", "ext_node", "fperm"):
            setattr(s, name, o[name].data_ptr())
        s.geo, s.fgeo, s.wu = self.geo.data_ptr(), self.fgeo.data_ptr(), self.wu.data_ptr()
        s.wp = self.wp.data_ptr() if self.wp is not None else None
        s.c2 = self.c2
        s.nbr, s.ncode = self.nbr.data_ptr(), self.ncode.data_ptr()
        s.halo = self.halo_buf.data_ptr() if self.halo_buf is not None else None
        s.n_halo = self.halo.n_recv if self.halo is not None else 0
        if self.minv_p is not None:
            s.minv_p, s.minv_u = self.minv_p.data_ptr(), self.minv_u.data_ptr()
        return s

    def with_formulation(self, strong_weak):
        s = _native.WadgProblem.from_buffer_copy(self.struct)
        s.formulation = _native.WADG_STRONG_WEAK if strong_weak else _native.WADG_STRONG
        return s

    # -- fields ----------------------------------------------------------------
    def empty_fields(self):
        return torch.zeros((self.fld, self.ref.Np, self.Kpad), dtype=self.dtype, device=self.device)

    @property
    def n_blocks(self):
        return self.Kpad // _native.ELEMS_PER_BLOCK

    def nbytes(self):
        tensors = [self.geo, self.fgeo, self.wu, self.nbr, self.ncode] + (
            [self.wp] if self.wp is not None else []) + (
            [self.minv_p, self.minv_u] if self.minv_p is not None else [])
        return sum(t.numel() * t.element_size() for t in tensors)
