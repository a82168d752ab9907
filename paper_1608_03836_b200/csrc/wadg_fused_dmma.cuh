// Fused LSRK45 stage for fp64 tetrahedra on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64).  Same algebra and data flow as k_stage_fused<double>
// (strong-weak volume, upwind/penalty surface, WADG update and LSRK axpy of
// R/pkg/src/wadg/solver.py:207-301, 348-363; one kernel per stage, Q
// ping-ponged), with every dense contraction a warp-level GEMM of 8 x 8 x 4
// DMMA tiles instead of DFMA register tiles:
//
//   D[e, n] (+)= sum_k A[e, k] B[k, n]      (e = element of the CTA, M)
//
// A = per-element data in shared memory, element fastest with a padded row
// stride KBS = KB + 4 doubles, so that the A fragment of a warp (element
// lane/4, row lane%4) is one conflict-free 64-bit load per lane.  B = a
// reference operator, packed on the host into fragment order
// [k step][n tile][lane] (device.dmma_operator_images) and staged by TMA bulk
// copies, so the B fragment is one contiguous 256-byte load.  One DMMA does
// 256 FMAs: the kernel issues ~8x fewer instructions than the DFMA tiles and
// the right-hand side R stays in registers (C-fragment layout) from the
// volume through the surface to the update.
//
// B200 measurements (profiles/r02_measured_peaks.json): DMMA 37.1 TFLOP/s,
// DFMA 34.1 TFLOP/s; the gain is in issue slots, registers and shared-memory
// traffic per FMA, which bound the DFMA kernel (ncu: FP64 pipe 33 % busy,
// short-scoreboard and barrier stalls, profiles/r02_ncu_stage_fused_f64_N4_c3.json).
#pragma once

namespace wadg {
namespace dk {

using fused::cdiv;
using fused::rup;

// SW: strong-weak form with the 2N+1 rules ((N+1)^3 volume, (N+1)^2 face
// points); otherwise the strong form with the sufficiency rules at N_geo = N
// (4N-3 volume: (2N-1)^3 points, 4N-2 face: (2N)^2 points; R/PAPER.md:288,294),
// the update always on the 2N+1 rule
template <int N, bool SW = true>
struct CfgD {
    static constexpr int NP = fused::np_tet(N);
    static constexpr int NPP = rup(NP, 8);                // nodes, padded to whole 8-wide tiles
    static constexpr int NKS = rup(NP, 4) / 4;            // k steps of a contraction over nodes (rows past NP are zero)
    static constexpr int NQ = SW ? (N + 1) * (N + 1) * (N + 1) : (2 * N - 1) * (2 * N - 1) * (2 * N - 1);
    static constexpr int NQU = (N + 1) * (N + 1) * (N + 1);
    static constexpr int NFP = fused::nfp_tri(N);
    static constexpr int NFPK = rup(NFP, 4);
    static constexpr int NFQ = SW ? (N + 1) * (N + 1) : 4 * N * N;
    static constexpr int NFQP = rup(NFQ, 8);
    static constexpr int NFKS = rup(NFQ, 4) / 4;           // k steps of the lift (face points past NFQ are zero)
    static constexpr int NF = 4, FLD = 4;
    // elements per CTA: 24 (three element tiles, six warps) for strong-weak N = 4,
    // so that two CTAs fit per SM (+1.5 %); 32 at N <= 5 otherwise; 16 at N = 6, 7
    // 16-element CTAs of four warps, four per SM, at strong-weak N = 2 (+3.7 % over
    // two 32-element CTAs; level at N = 3)
    static constexpr bool SMALL = SW && N == 2;
    static constexpr int KB = SMALL ? 16 : (SW && N == 4) ? 24 : ((N <= 5 && (SW || N <= 4)) ? 32 : 16);
    static constexpr int NW = KB == 24 ? 6 : (SMALL ? 4 : 8), NTH = 32 * NW;
    static constexpr int KBS = KB + 4;                     // shared row stride (doubles)
    static constexpr int MT = KB / 8;                      // element tiles
    static constexpr int WPM = NW / MT;                    // warps per element tile
    // quadrature points per chunk (32 for the strong form at N = 4, 5, so that
    // the four warps of an element tile each own a point tile)
    static constexpr int QC = (!SW && N >= 4) ? 32 : 16;
    static constexpr int NCH = cdiv(NQ, QC);               // volume chunks
    static constexpr int NCHU = cdiv(NQU, QC);             // update chunks
    static constexpr int NVA = SW ? 4 : 3;                 // operators of the point GEMM: D_a (and Vq)
    static constexpr int NVB = SW ? 4 : 1;                 // of the projection GEMM: DTW_a, -Pq (or -Pq)
    static constexpr int NWV = SW ? 6 : 4;                 // quadrature values per point: gp_i, F_a (or gp_i, div)
    static constexpr int QT = QC / 8;                      // point tiles per chunk
    static constexpr int JT = NPP / 8;                     // node tiles
    static constexpr int FT = NFQP / 8;                    // face-point tiles
    static constexpr int RT = cdiv(JT, WPM);               // R tiles per warp
    // two warps per element tile and an odd number of node tiles: the last node
    // tile is shared, fields 0, 1 to the first warp and 2, 3 to the second
    static constexpr bool SPLIT = WPM == 2 && JT % 2 == 1;
    static constexpr int AT = cdiv(QT, WPM);               // point tiles per warp (volume A, update z)
    // strong-weak point GEMMs split by group (D_a p | Vq u_i) where there are at
    // least twice as many warps per element tile as point tiles (N = 6, 7)
    static constexpr bool GSPLIT = SW && WPM >= 2 * QT;
    static constexpr int TT = cdiv(FT, WPM);               // face-point tiles per warp (traces)
    // operator images (doubles): [k step][n tile][32]
    static constexpr int IMG_VA = NVA * (NPP / 4) * QT * 32;   // D_r, D_s, D_t (, Vq) of one chunk
    static constexpr int IMG_VB = NVB * (QC / 4) * JT * 32;    // (DTW_r, DTW_s, DTW_t,) -Pq of one chunk
    static constexpr int IMG_VFI = (NFPK / 4) * FT * 32;
    static constexpr int IMG_LIFT = (NFQP / 4) * JT * 32;      // -Pf of one face
    static constexpr int IMG_U1 = (NPP / 4) * QT * 32;
    static constexpr int IMG_U2 = (QC / 4) * JT * 32;
    static constexpr size_t O_VA = 0;
    static constexpr size_t O_VB = O_VA + (size_t)NCH * IMG_VA;
    static constexpr size_t O_VFI = O_VB + (size_t)NCH * IMG_VB;
    static constexpr size_t O_LIFT = O_VFI + IMG_VFI;
    static constexpr size_t O_U1 = O_LIFT + (size_t)NF * IMG_LIFT;
    static constexpr size_t O_U2 = O_U1 + (size_t)NCHU * IMG_U1;
    static constexpr size_t OP_TOTAL = O_U2 + (size_t)NCHU * IMG_U2;
    // shared memory (bytes)
    static constexpr size_t SQ = (size_t)FLD * NPP * KBS * 8;
    static constexpr size_t PH_V = ((size_t)IMG_VA + IMG_VB + (size_t)NWV * QC * KBS) * 8;
    static constexpr size_t S_P1 = (size_t)FLD * NFPK * KBS * 8;
    // double-buffered neighbour face nodes (single at N = 7 to fit; single for the
    // strong form at N = 3, which would fit two CTAs per SM, was 3 % slower)
    static constexpr bool DBLP = N <= 6;
    static constexpr size_t S_TAB = (size_t)rup(2 * NF * KB + NF * NFP + NF * 6 * NFP + 6 * NFP, 4) * 4;
    static constexpr size_t PH_S = (DBLP ? 2 : 1) * S_P1 + ((size_t)FLD * NFQP * KBS + IMG_VFI + IMG_LIFT) * 8 + S_TAB;
    static constexpr size_t PH_U = ((size_t)FLD * NPP * KBS + IMG_U1 + IMG_U2 + (size_t)FLD * QC * KBS) * 8;
    static constexpr size_t PH = fused::maxz(PH_V, fused::maxz(PH_S, PH_U));
    static constexpr size_t SMEM = 16 + SQ + PH;
    // two CTAs per SM where they fit (<= 113 KB of shared memory; registers then
    // capped by the launch bounds): N = 3 12.5 -> 16.8 GDOF/s
    static constexpr int MINB = (SMALL && SMEM <= 56 * 1024) ? 4 : SMEM <= 113 * 1024 ? 2 : 1;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

// A fragment of element tile mt, k step ks from an element-fastest array
// (row k at x + k * KBS): lane holds A[e = 8 mt + lane/4][k = 4 ks + lane%4]
template <int KBS>
__device__ __forceinline__ double afrag(const double *x, int mt, int ks, int lane) {
    return x[(4 * ks + (lane & 3)) * KBS + 8 * mt + (lane >> 2)];
}

template <int N, bool SW>
__global__ void __launch_bounds__(CfgD<N, SW>::NTH, CfgD<N, SW>::MINB)
k_stage_dmma(const fused::FProb<double> P, const double *__restrict__ Qin, double *__restrict__ Qout,
             double *__restrict__ res, double tau_p, double tau_u, double a_rk, double b_rk, double dt, int block0) {
    using C = CfgD<N, SW>;
    constexpr int NP = C::NP, NPP = C::NPP, NQ = C::NQ, NQU = C::NQU, NFP = C::NFP, NFPK = C::NFPK, NFQ = C::NFQ;
    constexpr int NFQP = C::NFQP, NF = 4, FLD = 4, KB = C::KB, KBS = C::KBS, MT = C::MT, WPM = C::WPM;
    constexpr int QC = C::QC, QT = C::QT, JT = C::JT, FT = C::FT, RT = C::RT, AT = C::AT, TT = C::TT;
    constexpr bool SPLIT = C::SPLIT;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    double *sQ = reinterpret_cast<double *>(smem_raw + 16);
    double *ph = sQ + (size_t)FLD * NPP * KBS;
    // volume
    double *sVA = ph, *sVB = sVA + C::IMG_VA, *sW = sVB + C::IMG_VB;           // sW: [NWV][QC][KBS]
    // surface
    double *sP = ph;                                                           // [1 or 2][FLD][NFPK][KBS]
    double *sG = sP + (C::DBLP ? 2 : 1) * FLD * NFPK * KBS;                    // [FLD][NFQP][KBS]
    double *sVfi = sG + FLD * NFQP * KBS;
    double *sLift = sVfi + C::IMG_VFI;
    int32_t *sNbr = reinterpret_cast<int32_t *>(sLift + C::IMG_LIFT);
    int32_t *sCode = sNbr + NF * KB;
    int32_t *sFmask = sCode + NF * KB;
    int32_t *sExt = sFmask + NF * NFP;
    int32_t *sPerm = sExt + NF * 6 * NFP;
    // update
    double *sR = ph;                                                           // [FLD][NPP][KBS]
    double *sU1 = sR + FLD * NPP * KBS, *sU2 = sU1 + C::IMG_U1, *sW2 = sU2 + C::IMG_U2;   // sW2: [FLD][QC][KBS]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int mt = warp % MT, w0 = warp / MT;                 // element tile; first n tile of this warp
    const int er = lane >> 2, ec = 2 * (lane & 3);            // C fragment: element row, first column
    const int e = 8 * mt + er;                                // this lane's element (C fragments)
    // R tiles of this warp: node tile rjt(t) (valid if < JT), field c if rfld(t, c)
    auto rjt = [&](int t) { return (SPLIT && t == RT - 1) ? JT - 1 : w0 + WPM * t; };
    auto rfld = [&](int t, int c) { return !(SPLIT && t == RT - 1) || (c >> 1) == w0; };
    const size_t S = P.Kpad;
    const size_t kblk = (size_t)(block0 + blockIdx.x) * KB;
    const double *ops = P.opVA;

    WADG_PROF_MARK(0);
    if (tid == 0) {
        fused::mbar_init(&bar[0], 1);    // "A" operator images (VA, Vfi / Pf, Vu)
        fused::mbar_init(&bar[1], 1);    // "B" operator images (VB, Pu)
    }
    uint32_t pa = 0, pb = 0;             // phases of bar[0], bar[1]
    auto tma = [&](int k, double *dst, const double *src, int n) {   // thread 0 issues
        if (tid == 0) {
            fused::fence_proxy_async();
            fused::mbar_expect_tx(&bar[k], (uint32_t)(n * 8));
            fused::bulk_g2s(dst, src, (uint32_t)(n * 8), &bar[k]);
        }
    };
    auto twait = [&](int k) {
        uint32_t &ph = k ? pb : pa;
        fused::mbar_wait(&bar[k], ph);
        ph ^= 1u;
    };
    // chunk 0's volume operators land while the fields are staged
    tma(0, sVA, ops + C::O_VA, C::IMG_VA);
    tma(1, sVB, ops + C::O_VB, C::IMG_VB);
    // ---- fields -> sQ[c][j][e] (rows NP..NPP-1 zero) ------------------------
    for (int r = tid; r < FLD * NPP * (KB / 2); r += C::NTH) {
        const int e2 = (r % (KB / 2)) * 2, row = r / (KB / 2);
        const int c = row / NPP, j = row % NPP;
        double *dst = sQ + row * KBS + e2;
        if (j < NP)
            fused::cp_async16(dst, Qin + (size_t)(c * NP + j) * S + kblk + e2);
        else
            dst[0] = dst[1] = 0.0;
    }
    fused::cp_async_commit();
    fused::cp_async_wait<0>();
    // R accumulators (C fragments): field c, node tile jt = w0 + WPM * t
    double acc[RT][FLD][2];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
        for (int c = 0; c < FLD; ++c) acc[t][c][0] = acc[t][c][1] = 0.0;
    __syncthreads();
    WADG_PROF_MARK(1);

    // ======================= volume =======================================
    // operator images double as a pipeline: VA(ch+1) loads during phase B(ch),
    // VB(ch+1) during phase A(ch+1); chunk 0's were issued before the fields
    for (int ch = 0; ch < C::NCH; ++ch) {
        twait(0);
        if constexpr (!SW) {
            // strong form: du_a,c = D_a Q_c for all four fields; gp_i = sum_a G_ai du_a,0,
            // div = sum_i sum_a G_ai du_a,i (R/pkg/src/wadg/solver.py:259-264)
            double G[AT][2][9];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = ch * QC + 8 * (w0 + WPM * t) + ec + h;
                    const bool ok = w0 + WPM * t < QT && q < NQ;
#pragma unroll
                    for (int r = 0; r < 9; ++r)
                        G[t][h][r] = ok ? __ldg(P.geo + (size_t)(r * NQ + q) * S + kblk + e) : 0.0;
                }
            double d[AT][3][FLD][2];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int c = 0; c < FLD; ++c) d[t][a][c][0] = d[t][a][c][1] = 0.0;
#pragma unroll 2
            for (int ks = 0; ks < C::NKS; ++ks) {
                double x[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) x[c] = afrag<KBS>(sQ + c * NPP * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < AT; ++t) {
                    const int qt = w0 + WPM * t;
                    if (qt < QT) {
#pragma unroll
                        for (int a = 0; a < 3; ++a) {
                            const double b = sVA[((a * (NPP / 4) + ks) * QT + qt) * 32 + lane];
#pragma unroll
                            for (int c = 0; c < FLD; ++c) dmma(d[t][a][c], x[c], b);
                        }
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < AT; ++t) {
                const int qt = w0 + WPM * t;
                if (qt < QT) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int qq = 8 * qt + ec + h;
                        const double *g = G[t][h];
                        double div = 0.0;
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            sW[(i * QC + qq) * KBS + e] =
                                g[0 * 3 + i] * d[t][0][0][h] + g[1 * 3 + i] * d[t][1][0][h] + g[2 * 3 + i] * d[t][2][0][h];
                            div += g[0 * 3 + i] * d[t][0][1 + i][h] + g[1 * 3 + i] * d[t][1][1 + i][h] +
                                   g[2 * 3 + i] * d[t][2][1 + i][h];
                        }
                        sW[(3 * QC + qq) * KBS + e] = div;
                    }
                }
            }
        } else
        if constexpr (C::GSPLIT) {
            // A, one (point tile, group) unit per warp: group 0 dp_a = D_a p -> gp_i,
            // group 1 U_i = Vq u_i -> F_a (N = 6, 7: 2.x point tiles per four warps)
            const int qt = w0 % QT, grp = w0 / QT;
            if (grp < 2) {
                double G[2][9];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = ch * QC + 8 * qt + ec + h;
#pragma unroll
                    for (int r = 0; r < 9; ++r) G[h][r] = q < NQ ? __ldg(P.geo + (size_t)(r * NQ + q) * S + kblk + e) : 0.0;
                }
                double d[3][2];
#pragma unroll
                for (int m = 0; m < 3; ++m) d[m][0] = d[m][1] = 0.0;
                if (grp == 0) {
#pragma unroll 2
                    for (int ks = 0; ks < C::NKS; ++ks) {
                        const double x = afrag<KBS>(sQ, mt, ks, lane);
#pragma unroll
                        for (int m = 0; m < 3; ++m) dmma(d[m], x, sVA[((m * (NPP / 4) + ks) * QT + qt) * 32 + lane]);
                    }
                } else {
#pragma unroll 2
                    for (int ks = 0; ks < C::NKS; ++ks) {
                        const double b = sVA[((3 * (NPP / 4) + ks) * QT + qt) * 32 + lane];
#pragma unroll
                        for (int i = 0; i < 3; ++i) dmma(d[i], afrag<KBS>(sQ + (1 + i) * NPP * KBS, mt, ks, lane), b);
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int qq = 8 * qt + ec + h;
                    const double *g = G[h];
                    if (grp == 0) {
#pragma unroll
                        for (int i = 0; i < 3; ++i)
                            sW[(i * QC + qq) * KBS + e] = g[0 * 3 + i] * d[0][h] + g[1 * 3 + i] * d[1][h] + g[2 * 3 + i] * d[2][h];
                    } else {
#pragma unroll
                        for (int a = 0; a < 3; ++a)
                            sW[((3 + a) * QC + qq) * KBS + e] = g[a * 3 + 0] * d[0][h] + g[a * 3 + 1] * d[1][h] +
                                                                g[a * 3 + 2] * d[2][h];
                    }
                }
            }
        } else
        // A: dp_a = D_a p (m = 0..2), U_i = Vq u_i (m = 3..5) at the chunk's points; all
        // point tiles of this warp share the field fragments of a k step.  The
        // epilogue's geometric factors are loaded first, so their latency overlaps
        // the MMAs.
        {
            double G[AT][2][9];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = ch * QC + 8 * (w0 + WPM * t) + ec + h;
                    const bool ok = w0 + WPM * t < QT && q < NQ;
#pragma unroll
                    for (int r = 0; r < 9; ++r)
                        G[t][h][r] = ok ? __ldg(P.geo + (size_t)(r * NQ + q) * S + kblk + e) : 0.0;
                }
            double d[AT][6][2];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int m = 0; m < 6; ++m) d[t][m][0] = d[t][m][1] = 0.0;
#pragma unroll 2
            for (int ks = 0; ks < C::NKS; ++ks) {
                double x[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) x[c] = afrag<KBS>(sQ + c * NPP * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < AT; ++t) {
                    const int qt = w0 + WPM * t;
                    if (qt < QT) {
                        double b[4];
#pragma unroll
                        for (int m = 0; m < 4; ++m) b[m] = sVA[((m * (NPP / 4) + ks) * QT + qt) * 32 + lane];
#pragma unroll
                        for (int m = 0; m < 3; ++m) dmma(d[t][m], x[0], b[m]);
#pragma unroll
                        for (int i = 0; i < 3; ++i) dmma(d[t][3 + i], x[1 + i], b[3]);
                    }
                }
            }
            // epilogue: gp_i = sum_a G_ai dp_a, F_a = sum_i G_ai U_i (w is folded into DTW)
#pragma unroll
            for (int t = 0; t < AT; ++t) {
                const int qt = w0 + WPM * t;
                if (qt < QT) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int qq = 8 * qt + ec + h;
                        const double *g = G[t][h];
#pragma unroll
                        for (int i = 0; i < 3; ++i)
                            sW[(i * QC + qq) * KBS + e] = g[0 * 3 + i] * d[t][0][h] + g[1 * 3 + i] * d[t][1][h] +
                                                          g[2 * 3 + i] * d[t][2][h];
#pragma unroll
                        for (int a = 0; a < 3; ++a)
                            sW[((3 + a) * QC + qq) * KBS + e] = g[a * 3 + 0] * d[t][3][h] + g[a * 3 + 1] * d[t][4][h] +
                                                                g[a * 3 + 2] * d[t][5][h];
                    }
                }
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCH) tma(0, sVA, ops + C::O_VA + (size_t)(ch + 1) * C::IMG_VA, C::IMG_VA);
        twait(1);
        // B: R_p += sum_a DTW_a F_a (strong: (-Pq) div), R_u_i += (-Pq) gp_i
        if constexpr (!SW) {
#pragma unroll 2
            for (int ks = 0; ks < QC / 4; ++ks) {
                double w[4];
#pragma unroll
                for (int m = 0; m < 4; ++m) w[m] = afrag<KBS>(sW + m * QC * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int jt = rjt(t);
                    if (jt < JT) {
                        const double b = sVB[(ks * JT + jt) * 32 + lane];
                        if (rfld(t, 0)) dmma(acc[t][0], w[3], b);
#pragma unroll
                        for (int i = 0; i < 3; ++i)
                            if (rfld(t, 1 + i)) dmma(acc[t][1 + i], w[i], b);
                    }
                }
            }
        } else
#pragma unroll 4   // QC / 4 = 4 k steps: fully unrolled (with the lift and R' loops, +1 to +2.7 % at N = 2..7)
        for (int ks = 0; ks < QC / 4; ++ks) {
            double w[6];
#pragma unroll
            for (int m = 0; m < 6; ++m) w[m] = afrag<KBS>(sW + m * QC * KBS, mt, ks, lane);
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int jt = rjt(t);
                if (jt < JT) {
                    double b[4];
#pragma unroll
                    for (int m = 0; m < 4; ++m) b[m] = sVB[((m * (QC / 4) + ks) * JT + jt) * 32 + lane];
                    if (rfld(t, 0)) {
#pragma unroll
                        for (int a = 0; a < 3; ++a) dmma(acc[t][0], w[3 + a], b[a]);
                    }
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        if (rfld(t, 1 + i)) dmma(acc[t][1 + i], w[i], b[3]);
                }
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCH) tma(1, sVB, ops + C::O_VB + (size_t)(ch + 1) * C::IMG_VB, C::IMG_VB);
    }

    // ======================= surface ======================================
    const int NFQT = NF * NFQ;
    __syncthreads();
    WADG_PROF_MARK(2);
    for (int r = tid; r < NF * KB; r += C::NTH) {
        const int f = r / KB, el = r % KB;
        sNbr[r] = P.nbr[(size_t)f * S + kblk + el];
        sCode[r] = P.ncode[(size_t)f * S + kblk + el];
    }
    for (int r = tid; r < NF * NFP; r += C::NTH) sFmask[r] = __ldg(P.fmask + r);
    for (int r = tid; r < NF * 6 * NFP; r += C::NTH) sExt[r] = __ldg(P.ext_node + r);
    for (int r = tid; r < 6 * NFP; r += C::NTH) sPerm[r] = __ldg(P.fperm + r);
    // the Vfi image stays for the whole surface
    tma(0, sVfi, ops + C::O_VFI, C::IMG_VFI);
    twait(0);
    __syncthreads();
    // exterior face-node values of face f -> buf[c][i][e] (rows NFP..NFPK-1 zero)
    // NTH is a multiple of KB, so a thread's element is fixed: its neighbour,
    // orientation code and their table rows are read once per face (with the
    // weight prefetch below: N = 2 / 3 +3.7 / +2.2 %, N = 4, 5 level)
    static_assert(C::NTH % KB == 0, "gather assumes whole element rows per thread group");
    auto gather = [&](int f, double *buf) {
        const int el = tid % KB;
        const int nb = sNbr[f * KB + el], code = sCode[f * KB + el];
        const int32_t *ext = sExt + code * NFP;
#pragma unroll 2
        for (int rest = tid / KB; rest < FLD * NFPK; rest += C::NTH / KB) {
            const int i = rest % NFPK, c = rest / NFPK;
            double *dst = buf + rest * KBS + el;
            if (i >= NFP) {
                *dst = 0.0;
            } else if (nb >= 0) {
                fused::cp_async_elem(dst, Qin + (size_t)(c * NP + ext[i]) * S + nb);
            } else if (nb == -1) {       // mirror BC (solver.py:214-217): p+ = -p-, u+ = u-
                const double m = sQ[(c * NPP + sFmask[f * NFP + i]) * KBS + el];
                *dst = (c == 0) ? -m : m;
            } else {
                fused::cp_async_elem(dst, P.halo + ((size_t)(-nb - 2) * FLD + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
            }
        }
        fused::cp_async_commit();
    };
    gather(0, sP);
    for (int f = 0; f < NF; ++f) {
        double *cur = C::DBLP ? sP + (f & 1) * (FLD * NFPK * KBS) : sP;
        if (C::DBLP && f + 1 < NF) {
            gather(f + 1, sP + ((f + 1) & 1) * (FLD * NFPK * KBS));
            fused::cp_async_wait<1>();
        } else {
            fused::cp_async_wait<0>();   // single buffer: face f's nodes were gathered during face f-1's lift
        }
        tma(0, sLift, ops + C::O_LIFT + (size_t)f * C::IMG_LIFT, C::IMG_LIFT);   // lands during the traces
        __syncthreads();
        // traces at the face points: own (face nodes of sQ) and exterior (cur), then
        // the flux; the face factors are loaded before the MMAs
        {
            double fgv[TT][2][4];
#pragma unroll
            for (int t = 0; t < TT; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int fq = 8 * (w0 + WPM * t) + ec + h;
                    const bool ok = w0 + WPM * t < FT && fq < NFQ;
                    const size_t o = (size_t)(f * NFQ + fq) * S + kblk + e;
#pragma unroll
                    for (int dd = 0; dd < 4; ++dd) fgv[t][h][dd] = ok ? __ldg(P.fgeo + (size_t)dd * NFQT * S + o) : 0.0;
                }
            double dm[TT][FLD][2], dpv[TT][FLD][2];
#pragma unroll
            for (int t = 0; t < TT; ++t)
#pragma unroll
                for (int c = 0; c < FLD; ++c) dm[t][c][0] = dm[t][c][1] = dpv[t][c][0] = dpv[t][c][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < NFPK / 4; ++ks) {
                const int i = 4 * ks + (lane & 3);
                const int node = i < NFP ? sFmask[f * NFP + i] : -1;
                double xm[FLD], xp[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    xm[c] = node >= 0 ? sQ[(c * NPP + node) * KBS + 8 * mt + (lane >> 2)] : 0.0;
                    xp[c] = cur[(c * NFPK + i) * KBS + 8 * mt + (lane >> 2)];
                }
#pragma unroll
                for (int t = 0; t < TT; ++t) {
                    const int ft = w0 + WPM * t;
                    if (ft < FT) {
                        const double b = sVfi[(ks * FT + ft) * 32 + lane];
#pragma unroll
                        for (int c = 0; c < FLD; ++c) {
                            dmma(dm[t][c], xm[c], b);
                            dmma(dpv[t][c], xp[c], b);
                        }
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < TT; ++t) {
                const int ft = w0 + WPM * t;
                if (ft < FT) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int fq = 8 * ft + ec + h;
                        const double n0 = fgv[t][h][0], n1 = fgv[t][h][1], n2 = fgv[t][h][2], sJh = fgv[t][h][3];
                        const double djp = dpv[t][0][h] - dm[t][0][h];
                        const double dUn = (dpv[t][1][h] - dm[t][1][h]) * n0 + (dpv[t][2][h] - dm[t][2][h]) * n1 +
                                           (dpv[t][3][h] - dm[t][3][h]) * n2;
                        const double avg = (dpv[t][1][h] + dm[t][1][h]) * n0 + (dpv[t][2][h] + dm[t][2][h]) * n1 +
                                           (dpv[t][3][h] + dm[t][3][h]) * n2;
                        const double fpp = (SW ? avg : dUn) - tau_p * djp;   // strong: [u.n] (solver.py:220-232)
                        const double fuu = djp - tau_u * dUn;
                        // padded face points have zero factors, hence zero flux
                        sG[(0 * NFQP + fq) * KBS + e] = fpp * sJh;
                        sG[(1 * NFQP + fq) * KBS + e] = fuu * (sJh * n0);
                        sG[(2 * NFQP + fq) * KBS + e] = fuu * (sJh * n1);
                        sG[(3 * NFQP + fq) * KBS + e] = fuu * (sJh * n2);
                    }
                }
            }
        }
        __syncthreads();
        if (!C::DBLP && f + 1 < NF) gather(f + 1, sP);   // the traces are done with the buffer
        // L2 prefetch of the next face's factors, loaded before its trace MMAs
        if (f + 1 < NF)
            for (int r = tid; r < 4 * NFQ; r += C::NTH) {
                const double *p = P.fgeo + (size_t)(r / NFQ) * NFQT * S + (size_t)((f + 1) * NFQ + r % NFQ) * S + kblk;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p + KB - 1));
            }
        twait(0);
        // lift: R_c += (-Pf_f) g_c
#pragma unroll (C::NFKS % 3 == 0 ? 3 : 2)
        for (int ks = 0; ks < C::NFKS; ++ks) {
            double gv[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) gv[c] = afrag<KBS>(sG + c * NFQP * KBS, mt, ks, lane);
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int jt = rjt(t);
                if (jt < JT) {
                    const double b = sLift[(ks * JT + jt) * 32 + lane];
#pragma unroll
                    for (int c = 0; c < FLD; ++c)
                        if (rfld(t, c)) dmma(acc[t][c], gv[c], b);
                }
            }
        }
        __syncthreads();
    }

    // ======================= WADG update + LSRK ===========================
    WADG_PROF_MARK(3);
    // R -> sR[c][j][e] (the A operand of z = Vu R); accumulators restart at zero
    // L2 prefetch of this tile's old res rows, read by the LSRK write after the
    // update (N = 2 / 3 / 4: +1.2 / +0.5 / +2.3 % with the face-factor prefetch)
    if (a_rk != 0.0)
        for (int r = tid; r < FLD * NP; r += C::NTH) {
            const double *p = res + (size_t)r * S + kblk;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p + KB - 1));
        }
    // and of the update weights (c^2/J, 1/J), loaded before each chunk's MMAs
    for (int r = tid; r < 2 * NQU; r += C::NTH) {
        const double *w = r < NQU ? P.wu : P.wp;
        if (w) {
            const double *p = w + (size_t)(r % NQU) * S + kblk;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(p + KB - 1));
        }
    }
    tma(0, sU1, ops + C::O_U1, C::IMG_U1);
    tma(1, sU2, ops + C::O_U2, C::IMG_U2);
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int jt = rjt(t);
        if (jt < JT) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                if (rfld(t, c)) {
                    sR[(c * NPP + 8 * jt + ec) * KBS + e] = acc[t][c][0];
                    sR[(c * NPP + 8 * jt + ec + 1) * KBS + e] = acc[t][c][1];
                }
                acc[t][c][0] = acc[t][c][1] = 0.0;
            }
        }
    }
    __syncthreads();
    for (int ch = 0; ch < C::NCHU; ++ch) {
        twait(0);
        // z_c = Vu R_c at the chunk's points, times c^2/J (p) or 1/J (u); the weights
        // are loaded before the MMAs
        {
            double wu[AT][2], wp[AT][2];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int q = ch * QC + 8 * (w0 + WPM * t) + ec + h;
                    const bool ok = w0 + WPM * t < QT && q < NQU;
                    wu[t][h] = ok ? __ldg(P.wu + (size_t)q * S + kblk + e) : 0.0;
                    wp[t][h] = (ok && P.wp) ? __ldg(P.wp + (size_t)q * S + kblk + e) : 0.0;   // c^2 wu if no wp
                }
            double z[AT][FLD][2];
#pragma unroll
            for (int t = 0; t < AT; ++t)
#pragma unroll
                for (int c = 0; c < FLD; ++c) z[t][c][0] = z[t][c][1] = 0.0;
#pragma unroll (N >= 6 ? 3 : 2)   // z = Vu R: NKS = 21, 30 at N = 6, 7 (+1.7 / +1.3 %)
            for (int ks = 0; ks < C::NKS; ++ks) {
                double x[FLD];
#pragma unroll
                for (int c = 0; c < FLD; ++c) x[c] = afrag<KBS>(sR + c * NPP * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < AT; ++t) {
                    const int qt = w0 + WPM * t;
                    if (qt < QT) {
                        const double b = sU1[(ks * QT + qt) * 32 + lane];
#pragma unroll
                        for (int c = 0; c < FLD; ++c) dmma(z[t][c], x[c], b);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < AT; ++t) {
                const int qt = w0 + WPM * t;
                if (qt < QT) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int qq = 8 * qt + ec + h;
                        sW2[(0 * QC + qq) * KBS + e] = (P.wp ? wp[t][h] : P.c2 * wu[t][h]) * z[t][0][h];
#pragma unroll
                        for (int c = 1; c < FLD; ++c) sW2[(c * QC + qq) * KBS + e] = wu[t][h] * z[t][c][h];
                    }
                }
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCHU) tma(0, sU1, ops + C::O_U1 + (size_t)(ch + 1) * C::IMG_U1, C::IMG_U1);
        twait(1);
        // R'_c += Pu (omega z_c)
#pragma unroll 4
        for (int ks = 0; ks < QC / 4; ++ks) {
            double wv[FLD];
#pragma unroll
            for (int c = 0; c < FLD; ++c) wv[c] = afrag<KBS>(sW2 + c * QC * KBS, mt, ks, lane);
#pragma unroll
            for (int t = 0; t < RT; ++t) {
                const int jt = rjt(t);
                if (jt < JT) {
                    const double b = sU2[(ks * JT + jt) * 32 + lane];
#pragma unroll
                    for (int c = 0; c < FLD; ++c)
                        if (rfld(t, c)) dmma(acc[t][c], wv[c], b);
                }
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCHU) tma(1, sU2, ops + C::O_U2 + (size_t)(ch + 1) * C::IMG_U2, C::IMG_U2);
    }
    WADG_PROF_MARK(4);
    // res = a res + dt Minv(rhs); Q_out = Q_in + b res  (this lane: element e, nodes ec, ec+1 of its tiles)
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int jt = rjt(t);
        if (jt < JT) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                if (!rfld(t, c)) continue;
                double rold[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 8 * jt + ec + h;
                    rold[h] = (a_rk != 0.0 && j < NP) ? __ldg(res + (size_t)(c * NP + j) * S + kblk + e) : 0.0;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = 8 * jt + ec + h;
                    if (j < NP) {
                        const size_t o = (size_t)(c * NP + j) * S + kblk + e;
                        const double r = a_rk * rold[h] + dt * acc[t][c][h];
                        res[o] = r;
                        Qout[o] = sQ[(c * NPP + j) * KBS + e] + b_rk * r;
                    }
                }
            }
        }
    }
    __syncthreads();
    WADG_PROF_MARK(5);
}

}  // namespace dk
}  // namespace wadg
