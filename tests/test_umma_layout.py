"""Host side of the tcgen05 fused stage (no GPU): the TF32 hi/lo split is exact
and the K-major no-swizzle tile image puts B[r, k] at the byte offset the
kernel's descriptors address (csrc/wadg_umma.cuh kmaj_off), and the packed
operator buffer has exactly the CfgU size."""

import numpy as np
import pytest

from paper_1608_03836_b200 import device, refelem


def test_tf32_split_is_exact_and_hi_is_tf32():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 1e3
    hi, lo = device.tf32_split(x)
    assert np.array_equal((hi.astype(np.float64) + lo.astype(np.float64)).astype(np.float32), x)
    assert np.all(hi.view(np.uint32) & np.uint32(0x1FFF) == 0)
    assert np.all(np.abs(lo) <= np.abs(x) * 2.0 ** -10)


@pytest.mark.parametrize("R,KT", [(16, 40), (48, 16), (64, 24), (32, 8)])
def test_kmajor_image_offsets(R, KT):
    B = np.arange(R * KT, dtype=np.float64).reshape(R, KT)
    img = device.kmajor_image(B)
    for r in range(R):
        for k in range(KT):
            off = (r // 8) * (KT // 4) * 128 + (k // 4) * 128 + (r % 8) * 16 + (k % 4) * 4
            assert img[off // 4] == B[r, k]


@pytest.mark.parametrize("N", [2, 3, 4])
def test_operator_image_size(N):
    ref = refelem.build_reference_element(N, refelem.ElementShape.Tetrahedron)
    rup = lambda a, b: -(-a // b) * b
    NP, NQ = ref.Np, ref.Nq
    NPK, NFPK = rup(NP, 8), rup(ref.nfp, 8)
    NPN = NPK
    NFH, NCH, NCHU = -(-ref.nfq // 16), -(-NQ // 16), -(-NQ // 16)
    cfg = dict(qc=16, nch=NCH, npp=NPK, qcs=NPN, njs=NFPK, nfq8=NFH)
    img = device.umma_operator_images(ref, ref, cfg)
    expect = (NCH * 2 * 48 * NPK + (-(-NCH // 2)) * 2 * 32 * NPK + NCH * 2 * 3 * NPN * 16 + NCH * 2 * NPN * 16
              + NFH * 2 * 16 * NFPK + 4 * NFH * 2 * NPN * 16 + NCHU * (2 * 16 * NPK + 2 * NPN * 16))
    assert img.size == expect and img.dtype == np.float32
    # first tile: D_r rows (quadrature points 0..15), hi + lo reproduce fp32(D_r)
    half = 48 * NPK
    t = (img[:half] + img[half:2 * half]).reshape(6, NPK // 4, 8, 4).transpose(0, 2, 1, 3).reshape(48, NPK)
    assert np.array_equal(t[:16, :NP], ref.Dq[0][:16].astype(np.float32))


def test_interleave_blocks_layout():
    import torch
    rows, npts, Kp = 3, 13, 256
    x = torch.arange(rows * npts * Kp, dtype=torch.float32).reshape(rows, npts, Kp)
    y = device.interleave_blocks(x, 16, 128)
    assert y.shape == (2, rows, 4, 128, 4)
    for b, r, q, e in [(0, 0, 0, 0), (1, 2, 12, 127), (0, 1, 7, 33), (1, 0, 5, 64)]:
        assert y[b, r, q // 4, e, q % 4] == x[r, q, b * 128 + e]
    assert torch.all(y[:, :, 3, :, 1:] == 0)          # points 13..15 are zero padding


def test_dmma_fragment_images_reconstruct_operators():
    """The DMMA stage's B-fragment images (device.dmma_operator_images): lane t
    of [k step][n tile] holds B[4 ks + t % 4][8 nt + t // 4]; inverting that map
    must give back each operator (csrc/wadg_fused_dmma.cuh offsets)."""
    import numpy as np
    from paper_1608_03836_b200 import _native, device, refelem
    for N in (2, 4, 5):
        _native.call("wadg_debug_set_fused_variant", 3)
        try:
            cfg = _native.fused_config(_native.WADG_F64, N)
        finally:
            _native.call("wadg_debug_set_fused_variant", -1)
        assert cfg["kind"] == 3
        ref = refelem.build_reference_element(N, refelem.ElementShape.Tetrahedron)
        img = device.dmma_operator_images(ref, ref, cfg)
        QC, NCH, NPP, NFPK, NFQP = cfg["qc"], cfg["nch"], cfg["npp"], cfg["qcs"], cfg["njs"]

        def unpack(flat, K, Nn):
            a = flat.reshape(K // 4, Nn // 8, 32)
            B = np.zeros((K, Nn))
            for t in range(32):
                B[(4 * np.arange(K // 4))[:, None] + t % 4, (8 * np.arange(Nn // 8))[None, :] + t // 4] = a[:, :, t]
            return B
        o, NP, NQ = 0, ref.Np, ref.Nq
        sz = lambda K, Nn: K * Nn
        # last chunk of D_s (volume image VA): B[k=j][n=q] = Ds[ch QC + q, j]
        ch = NCH - 1
        o_va = (ch * 4 + 1) * sz(NPP, QC)
        B = unpack(img[o_va:o_va + sz(NPP, QC)], NPP, QC)
        q1 = NQ - ch * QC
        assert np.array_equal(B[:NP, :q1], ref.Dq[1][ch * QC:].T)
        assert not B[:, q1:].any()
        assert not B[NP:].any()
        # -Pq of chunk 0 (VB image, op 3): B[k=q][n=j] = -Pq[j, q]
        o_vb = NCH * 4 * sz(NPP, QC) + 3 * sz(QC, NPP)
        B = unpack(img[o_vb:o_vb + sz(QC, NPP)], QC, NPP)
        assert np.array_equal(B[:min(QC, NQ), :NP], -ref.Pq[:, :min(QC, NQ)].T)
        # -Pf of face 2: B[k=fq][n=j] = -Pf[j, 2 nfq + fq]
        o_l = NCH * 4 * sz(NPP, QC) + NCH * 4 * sz(QC, NPP) + sz(NFPK, NFQP) + 2 * sz(NFQP, NPP)
        B = unpack(img[o_l:o_l + sz(NFQP, NPP)], NFQP, NPP)
        nfq = ref.nfq
        assert np.array_equal(B[:nfq, :NP], -ref.Pfq[:, 2 * nfq:3 * nfq].T)
