// Fused LSRK45 stage for fp32 tetrahedra with tensor-core GEMM phases.
//
// Same dataflow as k_stage_fused (wadg_fused.cuh): one kernel per stage,
// ping-pong Q, neighbour face nodes by cp.async, operator chunks by TMA bulk
// copies, and the strong-weak volume, surface and WADG update/LSRK algebra of
// R/pkg/src/wadg/solver.py:207-301, 348-363.  The difference is that every
// dense contraction runs on the tensor cores as warp-level split-TF32 MMA
// (wadg_mma.cuh): x = hi + lo in registers, C += A_hi B_hi + A_hi B_lo +
// A_lo B_hi, so no extra shared memory holds split operands and the result
// keeps fp32 accuracy.
//
// A CTA owns KB = 64 elements = 4 MMA M-tiles of 16; the 8 warps are
// (M-tile) x (group), group 0 working on the pressure and group 1 on the
// velocity side of each phase, which balances the MMA counts:
//   volume A:  g0: dp_a = D_a p (3 B-operands), g1: U_i = Vq u_i (3 A-operands)
//   volume B:  g0: r_p += sum_a DTW_a F_a,      g1: r_u_i -= Pq gp_i
//   lift:      g0: r_p -= Pf_f g_p,             g1: r_u_i -= Pf_f g_u_i
//   update A:  g0: fields p, u1,  g1: u2, u3  (Vq, then the WADG weights)
//   update B:  same split, Pq
// Element-indexed shared arrays use a row stride of KB + 8 floats and the
// operator tiles strides = 8 (mod 32) so that every fragment load is
// bank-conflict free.

#pragma once

namespace wadg {
namespace tc {

using fused::cdiv;
using fused::rup;

__host__ __device__ constexpr int pad8mod32(int n) {   // smallest m >= n with m % 32 == 8
    return n + ((40 - (n % 32)) % 32);
}
__host__ __device__ constexpr int pad4mod32(int n) {   // smallest m >= n with m % 32 == 4
    return n + ((36 - (n % 32)) % 32);
}

template <int N>
struct CfgTC {
    static constexpr int NP = fused::np_tet(N);
    static constexpr int NPP = rup(NP, 8);                 // K extent over nodes (multiple of 8)
    static constexpr int NJT = NPP / 8;                    // N-tiles over nodes
    static constexpr int NJS = pad8mod32(NPP);             // row stride of [k][j] operator tiles
    static constexpr int NQ = (N + 1) * (N + 1) * (N + 1);
    static constexpr int NFP = fused::nfp_tri(N);
    static constexpr int NFQ = (N + 1) * (N + 1);
    static constexpr int NFQ8 = rup(NFQ, 8);
    static constexpr int NF = 4, FLD = 4;
    // 32 elements (2 MMA M-tiles) and 4 warps per CTA keep shared memory near
    // 106 KB so two independent CTAs share an SM and overlap each other's
    // barrier / memory phases
    static constexpr int KB = 32, MT = KB / 16;            // elements per CTA, M-tiles
    static constexpr int NTH = MT * 2 * 32;                 // (M-tile) x (group) warps
    static constexpr int QS = pad8mod32(KB);               // row stride of element-indexed arrays
    static constexpr int QC = 16, QCT = QC / 8;            // quadrature chunk, its N-tiles
    static constexpr int QCS = pad8mod32(QC);
    static constexpr int NCH = cdiv(NQ, QC);
    static constexpr size_t W = 4;
    static constexpr size_t SQ = (size_t)FLD * NPP * QS * W;
    // volume
    static constexpr size_t S_OPA = (size_t)4 * NPP * QCS * W;      // [m][j][QCS]
    static constexpr size_t S_OPB = (size_t)4 * QC * NJS * W;       // [m][q][NJS]
    static constexpr size_t S_W = (size_t)6 * QC * QS * W;          // [6][q][QS]
    static constexpr int GS = pad4mod32(KB);                       // row stride of prefetched factors
    static constexpr size_t S_GEO = (size_t)9 * QC * GS * W;        // [9][q][GS] geometric factors
    static constexpr size_t PH_V = S_OPA + S_OPB + S_W + S_GEO;
    // surface
    static constexpr int NFP8 = rup(NFP, 8);                       // K extent over face nodes
    static constexpr int NFQT8 = NFQ8 / 8;                         // N-tiles over face points
    static constexpr int VS = pad8mod32(NFQ8);                     // row stride of Vfi^T
    static constexpr size_t S_P1 = (size_t)FLD * NFP8 * QS * W;     // exterior face nodes [c][i][QS]
    static constexpr size_t S_TR = (size_t)2 * FLD * NFQ8 * QS * W; // traces [in|ex][c][fq][QS]
    static constexpr size_t S_FG = (size_t)4 * NFQ * QS * W;        // face factors [d][fq][QS]
    static constexpr size_t S_LIFT = (size_t)NFQ8 * NJS * W;        // [fq][NJS]
    static constexpr size_t S_VFI = (size_t)NFP8 * VS * W;          // Vfi^T [i][VS]
    static constexpr size_t S_TAB = (size_t)rup(2 * NF * KB + NF * NFP8 + NF * 6 * NFP + 6 * NFP, 4) * 4;
    // the flux g_c overwrites the interior traces in place (sG == sTr[0])
    static constexpr size_t PH_S = 2 * S_P1 + S_TR + S_FG + S_LIFT + S_VFI + S_TAB;
    // update
    static constexpr size_t S_R = SQ;
    static constexpr size_t S_U1 = (size_t)NPP * QCS * W;           // [j][QCS]
    static constexpr size_t S_U2 = (size_t)QC * NJS * W;            // [q][NJS]
    static constexpr size_t S_W2 = (size_t)FLD * QC * QS * W;
    static constexpr size_t S_OM = (size_t)2 * QC * GS * W;         // [wu|wp][q][GS]
    static constexpr size_t PH_U = S_R + S_U1 + S_U2 + S_W2 + S_OM;
    static constexpr size_t PH = fused::maxz(PH_V, fused::maxz(PH_S, PH_U));
    static constexpr size_t SMEM = 16 + SQ + PH;
};

template <int N>
__global__ void __launch_bounds__(CfgTC<N>::NTH, 2)
k_stage_fused_tc(const fused::FProb<float> P, const float *__restrict__ Qin, float *__restrict__ Qout,
                 float *__restrict__ res, float tau_p, float tau_u, float a_rk, float b_rk, float dt,
                 int block0) {
    using C = CfgTC<N>;
    using namespace fused;
    using namespace mma;
    constexpr int NP = C::NP, NPP = C::NPP, NJT = C::NJT, NJS = C::NJS, NQ = C::NQ;
    constexpr int NFP = C::NFP, NFQ = C::NFQ, NFQ8 = C::NFQ8, NF = C::NF, FLD = 4;
    constexpr int KB = C::KB, QS = C::QS, QC = C::QC, QCT = C::QCT, QCS = C::QCS;
    constexpr int FSQ = NPP * QS;                          // one field of sQ / sR
    constexpr int NTH = C::NTH, MT = C::MT;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    float *sQ = reinterpret_cast<float *>(smem_raw + 16);
    unsigned char *ph = smem_raw + 16 + C::SQ;
    float *sOpA = reinterpret_cast<float *>(ph);
    float *sOpB = reinterpret_cast<float *>(ph + C::S_OPA);
    float *sW = reinterpret_cast<float *>(ph + C::S_OPA + C::S_OPB);
    float *sGeo = reinterpret_cast<float *>(ph + C::S_OPA + C::S_OPB + C::S_W);
    float *sP = reinterpret_cast<float *>(ph);
    float *sTr = reinterpret_cast<float *>(ph + 2 * C::S_P1);
    float *sFG = reinterpret_cast<float *>(ph + 2 * C::S_P1 + C::S_TR);
    float *sG = sTr;                                   // [c][fq][QS], written over the interior traces
    float *sLift = reinterpret_cast<float *>(ph + 2 * C::S_P1 + C::S_TR + C::S_FG);
    float *sVfi = reinterpret_cast<float *>(ph + 2 * C::S_P1 + C::S_TR + C::S_FG + C::S_LIFT);
    int32_t *sNbr = reinterpret_cast<int32_t *>(ph + 2 * C::S_P1 + C::S_TR + C::S_FG + C::S_LIFT + C::S_VFI);
    int32_t *sCode = sNbr + NF * KB;
    int32_t *sFmask = sCode + NF * KB;               // [f][NFP8], padding -> a zero row of sQ
    int32_t *sExt = sFmask + NF * C::NFP8;
    int32_t *sPerm = sExt + NF * 6 * NFP;
    float *sR = reinterpret_cast<float *>(ph);
    float *sU1 = reinterpret_cast<float *>(ph + C::S_R);
    float *sU2 = reinterpret_cast<float *>(ph + C::S_R + C::S_U1);
    float *sW2 = reinterpret_cast<float *>(ph + C::S_R + C::S_U1 + C::S_U2);
    float *sOm = reinterpret_cast<float *>(ph + C::S_R + C::S_U1 + C::S_U2 + C::S_W2);
    constexpr int GS = C::GS;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int mt = warp % MT, grp = warp / MT;             // M-tile, pressure / velocity group
    const int e0 = mt * 16;
    const int g = lane >> 2, t = lane & 3;
    const size_t S = P.Kpad;
    const size_t kblk = (size_t)(block0 + blockIdx.x) * KB;
    WADG_PROF_MARK(0);

    if (tid == 0) mbar_init(bar, 1);
    // element fields via 16-byte cp.async, node rows >= NP zero
    for (int r = tid; r < FLD * NPP * (KB / 4); r += NTH) {
        const int e4 = (r % (KB / 4)) * 4, row = r / (KB / 4);
        const int c = row / NPP, j = row % NPP;
        float *dst = sQ + row * QS + e4;
        if (j < NP) {
            cp_async16(dst, Qin + (size_t)(c * NP + j) * S + kblk + e4);
        } else {
            dst[0] = dst[1] = dst[2] = dst[3] = 0.f;
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    BulkLoader ld{bar, 0u};
    __syncthreads();
    WADG_PROF_MARK(1);

    // persistent nodal accumulators (MMA C layout): group 0 -> r_p (1 field),
    // group 1 -> r_u (3 fields, stored with the opposite sign)
    float acc[3][NJT][4];
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int n = 0; n < NJT; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[f][n][i] = 0.f;

    // ======================= volume =======================================
    for (int ch = 0; ch < C::NCH; ++ch) {
        {   // geometric factors of this chunk: cp.async, overlapped with the MMAs below
            const int qn = min(QC, NQ - ch * QC);
            __syncthreads();                   // previous chunk's epilogue is done with sGeo
            for (int r = tid; r < 9 * qn * (KB / 4); r += NTH) {
                const int e4 = (r % (KB / 4)) * 4, row = r / (KB / 4);
                const int rr = row / qn, qq = row % qn;
                cp_async16(sGeo + (rr * QC + qq) * GS + e4, P.geo + (size_t)(rr * NQ + ch * QC + qq) * S + kblk + e4);
            }
            cp_async_commit();
        }
        ld.load2(sOpA, P.opVA + (size_t)ch * (C::S_OPA / 4), (uint32_t)C::S_OPA,
                 sOpB, P.opVB + (size_t)ch * (C::S_OPB / 4), (uint32_t)C::S_OPB);
        {
            // A: quadrature values of dp_a (g0) or U_i (g1) for this warp's 16 elements
            float c4[3][QCT][4];
#pragma unroll
            for (int m = 0; m < 3; ++m)
#pragma unroll
                for (int n = 0; n < QCT; ++n)
#pragma unroll
                    for (int i = 0; i < 4; ++i) c4[m][n][i] = 0.f;
#pragma unroll 2
            for (int k0 = 0; k0 < NPP; k0 += 8) {
                if (grp == 0) {
                    AFrag a;
                    load_a_colmajor(a, sQ + k0 * QS + e0, QS, lane);
                    BFrag b[3][QCT];
#pragma unroll
                    for (int m = 0; m < 3; ++m)
#pragma unroll
                        for (int n = 0; n < QCT; ++n) load_b_rowmajor(b[m][n], sOpA + (m * NPP + k0) * QCS + n * 8, QCS, lane);
                    mma3_aB<3, QCT>(c4, a, b);
                } else {
                    BFrag b[QCT];
#pragma unroll
                    for (int n = 0; n < QCT; ++n) load_b_rowmajor(b[n], sOpA + (3 * NPP + k0) * QCS + n * 8, QCS, lane);
                    AFrag a[3];
#pragma unroll
                    for (int m = 0; m < 3; ++m) load_a_colmajor(a[m], sQ + (1 + m) * FSQ + k0 * QS + e0, QS, lane);
                    mma3_AB<3, QCT>(c4, a, b);
                }
            }
            // pointwise geometric factors: g0 gp_i = sum_a G_ai dp_a, g1 F_a = sum_i G_ai U_i
            cp_async_wait<0>();
            __syncthreads();
#pragma unroll
            for (int n = 0; n < QCT; ++n)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int qq = n * 8 + 2 * t + (i & 1);
                    const int e = e0 + g + ((i >> 1) << 3);
                    const int q = ch * QC + qq;
                    float o[3] = {0.f, 0.f, 0.f};
                    if (q < NQ) {
                        float G[9];
#pragma unroll
                        for (int r = 0; r < 9; ++r) G[r] = sGeo[(r * QC + qq) * GS + e];
#pragma unroll
                        for (int m = 0; m < 3; ++m)
                            o[m] = (grp == 0) ? G[0 * 3 + m] * c4[0][n][i] + G[1 * 3 + m] * c4[1][n][i] + G[2 * 3 + m] * c4[2][n][i]
                                              : G[m * 3 + 0] * c4[0][n][i] + G[m * 3 + 1] * c4[1][n][i] + G[m * 3 + 2] * c4[2][n][i];
                    }
#pragma unroll
                    for (int m = 0; m < 3; ++m) sW[((grp * 3 + m) * QC + qq) * QS + e] = o[m];
                }
        }
        __syncthreads();
        // B: project to nodes with DTW_a (g0, from F_a) or Pq (g1, from gp_i)
#pragma unroll
        for (int k0 = 0; k0 < QC; k0 += 8) {
            if (grp == 0) {
                AFrag af[3];
                BFrag b[3][NJT];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    load_a_colmajor(af[a], sW + ((3 + a) * QC + k0) * QS + e0, QS, lane);
#pragma unroll
                    for (int n = 0; n < NJT; ++n) load_b_rowmajor(b[a][n], sOpB + (a * QC + k0) * NJS + n * 8, NJS, lane);
                }
                mma3_sum<3, NJT>(acc[0], af, b);
            } else {
                BFrag b[NJT];
#pragma unroll
                for (int n = 0; n < NJT; ++n) load_b_rowmajor(b[n], sOpB + (3 * QC + k0) * NJS + n * 8, NJS, lane);
                AFrag af[3];
#pragma unroll
                for (int m = 0; m < 3; ++m) load_a_colmajor(af[m], sW + (m * QC + k0) * QS + e0, QS, lane);
                mma3_AB<3, NJT>(acc, af, b);
            }
        }
    }

    // ======================= surface ======================================
    constexpr int NFP8 = C::NFP8, NFQT8 = C::NFQT8, VS = C::VS;
    const int NFQT = NF * NFQ;
    __syncthreads();
    WADG_PROF_MARK(2);
    for (int r = tid; r < NF * KB; r += NTH) {
        const int f = r / KB, e = r % KB;
        sNbr[r] = P.nbr[(size_t)f * S + kblk + e];
        sCode[r] = P.ncode[(size_t)f * S + kblk + e];
    }
    for (int r = tid; r < NF * NFP8; r += NTH) {
        const int f = r / NFP8, i = r % NFP8;
        sFmask[r] = i < NFP ? __ldg(P.fmask + f * NFP + i) : NP;     // row NP of sQ is zero padding
    }
    for (int r = tid; r < NF * 6 * NFP; r += NTH) sExt[r] = __ldg(P.ext_node + r);
    for (int r = tid; r < 6 * NFP; r += NTH) sPerm[r] = __ldg(P.fperm + r);
    for (int r = tid; r < NFP8 * VS; r += NTH) {                 // Vfi^T, zero padded
        const int i = r / VS, fq = r % VS;
        sVfi[r] = (i < NFP && fq < NFQ) ? __ldg(P.Vfi + fq * NFP + i) : 0.f;
    }
    if constexpr (NFP8 > NFP) {                                  // K-padding rows of both sP buffers
        constexpr int PADN = (NFP8 - NFP) * QS;
        for (int r = tid; r < 2 * FLD * PADN; r += NTH) {
            const int bc = r / PADN;                             // buffer * FLD + field
            sP[(bc * NFP8 + NFP) * QS + r % PADN] = 0.f;
        }
    }
    __syncthreads();
    auto gather = [&](int f, float *buf) {
        for (int r = tid; r < FLD * NFP * KB; r += NTH) {
            const int e = r % KB, rest = r / KB;
            const int i = rest % NFP, c = rest / NFP;
            const int nb = sNbr[f * KB + e];
            const int code = sCode[f * KB + e];
            float *dst = buf + (c * NFP8 + i) * QS + e;
            if (nb >= 0) {
                cp_async_elem(dst, Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nb);
            } else if (nb == -1) {
                const float m = sQ[(c * NPP + sFmask[f * NFP8 + i]) * QS + e];
                *dst = (c == 0) ? -m : m;
            } else {
                cp_async_elem(dst, P.halo + ((size_t)(-nb - 2) * FLD + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
            }
        }
    };
    gather(0, sP);
    cp_async_commit();
    for (int f = 0; f < NF; ++f) {
        float *cur = sP + (f & 1) * (FLD * NFP8 * QS);
        // this face's normals and sJ/2, then the next face's neighbour nodes
        for (int r = tid; r < 4 * NFQ * (KB / 4); r += NTH) {
            const int e4 = (r % (KB / 4)) * 4, row = r / (KB / 4);
            const int d = row / NFQ, fq = row % NFQ;
            cp_async16(sFG + row * QS + e4, P.fgeo + (size_t)(d * NFQT + f * NFQ + fq) * S + kblk + e4);
        }
        cp_async_commit();
        if (f + 1 < NF) {
            gather(f + 1, sP + ((f + 1) & 1) * (FLD * NFP8 * QS));
            cp_async_commit();
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, (uint32_t)C::S_LIFT);
            bulk_g2s(sLift, P.liftT + (size_t)f * NFQ8 * NJS, (uint32_t)C::S_LIFT, bar);
        }
        __syncthreads();
        // traces at face quadrature points on the tensor cores:
        // group 0 interior (face nodes of sQ via fmask), group 1 exterior (cur)
        {
            float tr[FLD][NFQT8][4];
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int n = 0; n < NFQT8; ++n)
#pragma unroll
                    for (int i = 0; i < 4; ++i) tr[c][n][i] = 0.f;
#pragma unroll
            for (int k0 = 0; k0 < NFP8; k0 += 8) {
                BFrag b[NFQT8];
#pragma unroll
                for (int n = 0; n < NFQT8; ++n) load_b_rowmajor(b[n], sVfi + k0 * VS + n * 8, VS, lane);
                const int r0 = (grp == 0) ? sFmask[f * NFP8 + k0 + t] : k0 + t;
                const int r1 = (grp == 0) ? sFmask[f * NFP8 + k0 + t + 4] : k0 + t + 4;
                AFrag af[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    const float *base = (grp == 0) ? sQ + c * FSQ : cur + c * NFP8 * QS;
                    const float *p0 = base + r0 * QS + e0 + g, *p1 = base + r1 * QS + e0 + g;
                    Split sp;
                    sp = split(p0[0]); af[c].hi[0] = sp.hi; af[c].lo[0] = sp.lo;
                    sp = split(p0[8]); af[c].hi[1] = sp.hi; af[c].lo[1] = sp.lo;
                    sp = split(p1[0]); af[c].hi[2] = sp.hi; af[c].lo[2] = sp.lo;
                    sp = split(p1[8]); af[c].hi[3] = sp.hi; af[c].lo[3] = sp.lo;
                }
                mma3_AB<FLD, NFQT8>(tr, af, b);
            }
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int n = 0; n < NFQT8; ++n)
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int fq = n * 8 + 2 * t + (i & 1);
                        const int e = e0 + g + ((i >> 1) << 3);
                        sTr[((grp * FLD + c) * NFQ8 + fq) * QS + e] = tr[c][n][i];
                    }
        }
        __syncthreads();
        // penalty flux, pointwise
        for (int r = tid; r < NFQ * KB; r += NTH) {
            const int e = r % KB, fq = r / KB;
            float mM[FLD], mP[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                mM[c] = sTr[((0 * FLD + c) * NFQ8 + fq) * QS + e];
                mP[c] = sTr[((1 * FLD + c) * NFQ8 + fq) * QS + e];
            }
            const float n0 = sFG[(0 * NFQ + fq) * QS + e], n1 = sFG[(1 * NFQ + fq) * QS + e];
            const float n2 = sFG[(2 * NFQ + fq) * QS + e], sJh = sFG[(3 * NFQ + fq) * QS + e];
            const float dp = mP[0] - mM[0];
            const float dUn = (mP[1] - mM[1]) * n0 + (mP[2] - mM[2]) * n1 + (mP[3] - mM[3]) * n2;
            const float avg = (mP[1] + mM[1]) * n0 + (mP[2] + mM[2]) * n1 + (mP[3] + mM[3]) * n2;
            const float fp = avg - tau_p * dp;
            const float fu = dp - tau_u * dUn;
            sG[(0 * NFQ8 + fq) * QS + e] = fp * sJh;
            sG[(1 * NFQ8 + fq) * QS + e] = fu * (sJh * n0);
            sG[(2 * NFQ8 + fq) * QS + e] = fu * (sJh * n1);
            sG[(3 * NFQ8 + fq) * QS + e] = fu * (sJh * n2);
        }
        __syncthreads();
        mbar_wait(bar, ld.phase);
        ld.phase ^= 1u;
        // lift: r_p -= Pf g_p (accumulated as + (-g_p)), r_u stored negated: += Pf g_u
#pragma unroll
        for (int k0 = 0; k0 < NFQ8; k0 += 8) {
            BFrag b[NJT];
#pragma unroll
            for (int n = 0; n < NJT; ++n) load_b_rowmajor(b[n], sLift + k0 * NJS + n * 8, NJS, lane);
            if (grp == 0) {
                AFrag af;
                load_a_colmajor(af, sG + k0 * QS + e0, QS, lane);
#pragma unroll
                for (int i = 0; i < 4; ++i) {    // negate: r_p -= Pf g_p
                    af.hi[i] ^= 0x80000000u;
                    af.lo[i] ^= 0x80000000u;
                }
                mma3_row<NJT>(acc[0], af, b);
            } else {
                AFrag af[3];
#pragma unroll
                for (int m = 0; m < 3; ++m) load_a_colmajor(af[m], sG + ((1 + m) * NFQ8 + k0) * QS + e0, QS, lane);
                mma3_AB<3, NJT>(acc, af, b);
            }
        }
        __syncthreads();
    }

    // ======================= WADG update + LSRK ===========================
    WADG_PROF_MARK(3);
    // rhs into sR: g0 writes r_p, g1 writes r_u = -acc
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        if (grp == 0 && m > 0) break;
        const int c = grp == 0 ? 0 : 1 + m;
        const float sg = grp == 0 ? 1.f : -1.f;
#pragma unroll
        for (int n = 0; n < NJT; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = n * 8 + 2 * t + (i & 1);
                const int e = e0 + g + ((i >> 1) << 3);
                sR[(c * NPP + j) * QS + e] = sg * acc[m][n][i];
                acc[m][n][i] = 0.f;
            }
    }
    // group 0 owns fields {0, 1}, group 1 fields {2, 3} in the update
    const int cf0 = grp * 2;
    for (int ch = 0; ch < C::NCH; ++ch) {
        {   // WADG weights of this chunk
            const int qn = min(QC, NQ - ch * QC);
            const int nw = P.wp ? 2 : 1;
            __syncthreads();
            for (int r = tid; r < nw * qn * (KB / 4); r += NTH) {
                const int e4 = (r % (KB / 4)) * 4, row = r / (KB / 4);
                const int w = row / qn, qq = row % qn;
                const float *src = (w == 0 ? P.wu : P.wp) + (size_t)(ch * QC + qq) * S + kblk + e4;
                cp_async16(sOm + (w * QC + qq) * GS + e4, src);
            }
            cp_async_commit();
        }
        ld.load2(sU1, P.opU1 + (size_t)ch * (C::S_U1 / 4), (uint32_t)C::S_U1,
                 sU2, P.opU2 + (size_t)ch * (C::S_U2 / 4), (uint32_t)C::S_U2);
        {
            float z[2][QCT][4];
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
                for (int n = 0; n < QCT; ++n)
#pragma unroll
                    for (int i = 0; i < 4; ++i) z[m][n][i] = 0.f;
#pragma unroll 2
            for (int k0 = 0; k0 < NPP; k0 += 8) {
                BFrag b[QCT];
#pragma unroll
                for (int n = 0; n < QCT; ++n) load_b_rowmajor(b[n], sU1 + k0 * QCS + n * 8, QCS, lane);
                AFrag af[2];
#pragma unroll
                for (int m = 0; m < 2; ++m) load_a_colmajor(af[m], sR + (cf0 + m) * FSQ + k0 * QS + e0, QS, lane);
                mma3_AB<2, QCT>(z, af, b);
            }
            cp_async_wait<0>();
            __syncthreads();
#pragma unroll
            for (int n = 0; n < QCT; ++n)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int qq = n * 8 + 2 * t + (i & 1);
                    const int e = e0 + g + ((i >> 1) << 3);
                    const int q = ch * QC + qq;
                    float wu = 0.f, wp = 0.f;
                    if (q < NQ) {
                        wu = sOm[qq * GS + e];
                        wp = P.wp ? sOm[(QC + qq) * GS + e] : P.c2 * wu;
                    }
#pragma unroll
                    for (int m = 0; m < 2; ++m)
                        sW2[((cf0 + m) * QC + qq) * QS + e] = ((cf0 + m) == 0 ? wp : wu) * z[m][n][i];
                }
        }
        __syncthreads();
#pragma unroll
        for (int k0 = 0; k0 < QC; k0 += 8) {
            BFrag b[NJT];
#pragma unroll
            for (int n = 0; n < NJT; ++n) load_b_rowmajor(b[n], sU2 + k0 * NJS + n * 8, NJS, lane);
            AFrag af[2];
#pragma unroll
            for (int m = 0; m < 2; ++m) load_a_colmajor(af[m], sW2 + ((cf0 + m) * QC + k0) * QS + e0, QS, lane);
            mma3_AB<2, NJT>(reinterpret_cast<float (&)[2][NJT][4]>(acc), af, b);
        }
    }
    __syncthreads();
    WADG_PROF_MARK(4);
    // res = a res + dt Minv(rhs); Q_out = Q_in + b res
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int c = cf0 + m;
#pragma unroll
        for (int n = 0; n < NJT; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int j = n * 8 + 2 * t + (i & 1);
                const int e = e0 + g + ((i >> 1) << 3);
                if (j < NP) {
                    const size_t o = (size_t)(c * NP + j) * S + kblk + e;
                    const float r = (a_rk == 0.f) ? dt * acc[m][n][i] : a_rk * res[o] + dt * acc[m][n][i];
                    res[o] = r;
                    Qout[o] = sQ[(c * NPP + j) * QS + e] + b_rk * r;
                }
            }
    }
    __syncthreads();
    WADG_PROF_MARK(5);
}

}  // namespace tc
}  // namespace wadg
