// Fused LSRK45 stage for fp32 tetrahedra at N >= 5 on the tensor cores, as
// warp-level split-TF32 mma.sync.m16n8k8 tiles.  Same algebra and data flow as
// the DMMA stage (csrc/wadg_fused_dmma.cuh; strong-weak volume, upwind/penalty
// surface, WADG update and LSRK axpy of R/pkg/src/wadg/solver.py:207-301,
// 348-363; one kernel per stage, Q ping-ponged):
//
//   D[e, n] (+)= sum_k A[e, k] B[k, n]      (e = element of the CTA, M = 16)
//
// * Why not tcgen05 here: at N = 5 the 128-element tcgen05 tile needs 229 KB of
//   shared memory for its fields and 224 TMEM columns for R alone (DESIGN.md
//   section 10).  These 16-element warp tiles keep R in registers, like the
//   DMMA stage, and fit two 32-element CTAs per SM.
// * fp32 accuracy: each product is A_lo B_hi + A_hi B_lo + A_hi B_hi with hi the
//   round-to-nearest tf32 part and lo the remainder (x = hi + lo to ~22 bits).
//   The tensor core's fp32 accumulation truncates (measured, scripts/hmma_bias.py: bias
//   -1.9e-6 after a K = 216 chain), so every k step of 8 accumulates into a
//   fresh fragment (C = 0) that is added to the running sum with an fp32 FADD:
//   bias -4.9e-8, independent of K.
// * Shared-memory layout of every A operand: element-fastest rows with the two
//   elements g and g + 8 of a 16-element tile adjacent (position 2g, 2g + 1),
//   row stride KBS = KB + 8 floats: an A fragment is two conflict-free 64-bit
//   loads per lane, and a C fragment's two rows are one 64-bit store.
// * B operands: reference operators packed on the host in fragment order
//   [k step][n tile][lane][hi(k=t), hi(k=t+4), lo(k=t), lo(k=t+4)]
//   (device.tmma_operator_images), one 128-bit load per fragment, staged by TMA
//   bulk copies.
#pragma once

namespace wadg {
namespace tk {

using fused::cdiv;
using fused::rup;

// SW: strong-weak form with the 2N+1 rules ((N+1)^3 volume, (N+1)^2 face
// points); otherwise the strong form with the sufficiency rules at N_geo = N
// ((2N-1)^3 volume, (2N)^2 face points; R/PAPER.md:288,294), as in the DMMA
// stage; the update always on the 2N+1 rule
template <int N, bool SW = true>
struct CfgT {
    static constexpr int NP = fused::np_tet(N);
    static constexpr int NPP = rup(NP, 8);
    static constexpr int NQ = SW ? (N + 1) * (N + 1) * (N + 1) : (2 * N - 1) * (2 * N - 1) * (2 * N - 1);
    static constexpr int NQU = (N + 1) * (N + 1) * (N + 1);
    static constexpr int NFP = fused::nfp_tri(N);
    static constexpr int NFPK = rup(NFP, 8);
    static constexpr int NFQ = SW ? (N + 1) * (N + 1) : 4 * N * N;
    static constexpr int NFQP = rup(NFQ, 8);
    static constexpr int NF = 4, FLD = 4;
    static constexpr int KB = 32;                          // elements per CTA: two 16-element tiles
    static constexpr int NW = 8, NTH = 32 * NW;
    static constexpr int KBS = KB + 8;                     // row stride (floats), = 8 mod 32
    static constexpr int MT = KB / 16;                     // element tiles
    static constexpr int WPM = NW / MT;                    // warps per element tile
    static constexpr int QC = 16;                          // quadrature points per chunk
    static constexpr int NCH = cdiv(NQ, QC), NCHU = cdiv(NQU, QC);
    static constexpr int QT = QC / 8, JT = NPP / 8, FT = NFQP / 8;
    static constexpr int RT = cdiv(JT, WPM);               // R node tiles per warp
    // point-GEMM units of the strong form: (point tile, field c: D_a Q_c)
    static constexpr int NAU = 4 * QT;
    static constexpr int AU = cdiv(NAU, WPM);
    static constexpr int NVA = SW ? 4 : 3;                 // operators of the point GEMM: D_a (, Vq)
    static constexpr int NVB = SW ? 4 : 1;                 // of the projection: (DTW_a,) -Pq
    static constexpr int NWR = SW ? 6 : 12;                // point-value rows of the volume (sW)
    // point-GEMM products (operator, point tile), in the order the warps of an
    // element tile take them: strong-weak (m, qt), m = D_r, D_s, D_t (on p), Vq (on
    // u1, u2, u3); strong (c, a, qt), D_a on field c
    static constexpr int NPROD = SW ? 6 * QT : 12 * QT;
    __host__ __device__ static constexpr int prod_qt(int P) { return P % QT; }
    __host__ __device__ static constexpr int prod_field(int P) { return SW ? (P / QT < 3 ? 0 : P / QT - 2) : P / (3 * QT); }
    __host__ __device__ static constexpr int prod_op(int P) { return SW ? (P / QT < 3 ? P / QT : 3) : (P / QT) % 3; }
    __host__ __device__ static constexpr int prod_row(int P) { return SW ? P / QT : 3 * (P / (3 * QT)) + (P / QT) % 3; }
    // number of products from P on (at most n) that share P's field
    __host__ __device__ static constexpr int prod_run(int P, int n) {
        int k = 0;
        while (k < n && prod_field(P + k) == prod_field(P)) ++k;
        return k;
    }
    static constexpr int TT = cdiv(FT, WPM);               // face-point tiles per warp
    static constexpr int ZU = cdiv(2 * QT, WPM);           // (point tile, field pair) units per warp
    static constexpr int FR = 128;                         // floats per fragment image (32 lanes x 4)
    static constexpr int IMG_VA = NVA * (NPP / 8) * QT * FR; // D_r, D_s, D_t (, Vq) of one chunk
    static constexpr int IMG_VB = NVB * (QC / 8) * JT * FR;  // (DTW_r, DTW_s, DTW_t,) -Pq of one chunk
    static constexpr int IMG_VFI = (NFPK / 8) * FT * FR;
    static constexpr int IMG_LIFT = (NFQP / 8) * JT * FR;  // -Pf of one face
    static constexpr int IMG_U1 = (NPP / 8) * QT * FR;
    static constexpr int IMG_U2 = (QC / 8) * JT * FR;
    static constexpr size_t O_VA = 0;
    static constexpr size_t O_VB = O_VA + (size_t)NCH * IMG_VA;
    static constexpr size_t O_VFI = O_VB + (size_t)NCH * IMG_VB;
    static constexpr size_t O_LIFT = O_VFI + IMG_VFI;
    static constexpr size_t O_U1 = O_LIFT + (size_t)NF * IMG_LIFT;
    static constexpr size_t O_U2 = O_U1 + (size_t)NCHU * IMG_U1;
    static constexpr size_t OP_TOTAL = O_U2 + (size_t)NCHU * IMG_U2;
    // shared memory (bytes)
    static constexpr size_t SQ = (size_t)FLD * NPP * KBS * 4;
    static constexpr size_t PH_V = ((size_t)IMG_VA + IMG_VB + (size_t)NWR * QC * KBS) * 4;
    static constexpr size_t S_P1 = (size_t)FLD * NFPK * KBS * 4;
    static constexpr size_t S_TAB = (size_t)rup(2 * NF * KB + NF * NFP + NF * 6 * NFP + 6 * NFP, 4) * 4;
    static constexpr size_t PH_S1 = ((size_t)FLD * NFQP * KBS + IMG_VFI + IMG_LIFT) * 4 + S_TAB;
    static constexpr size_t PH_U = ((size_t)FLD * NPP * KBS + IMG_U1 + IMG_U2 + (size_t)FLD * QC * KBS) * 4;
    static constexpr size_t PH_NOS = fused::maxz(PH_V, PH_U);
    // double-buffered neighbour face nodes only where two CTAs per SM still fit
    static constexpr bool DBLP = 16 + SQ + fused::maxz(PH_NOS, 2 * S_P1 + PH_S1) <= 113 * 1024;
    static constexpr size_t PH_S = (DBLP ? 2 : 1) * S_P1 + PH_S1;
    static constexpr size_t PH = fused::maxz(PH_NOS, PH_S);
    static constexpr size_t SMEM = 16 + SQ + PH;
    static constexpr int MINB = SMEM <= 113 * 1024 ? 2 : 1;
};

// x = hi + lo with hi = x rounded to the nearest tf32 (ties away, as
// device.tf32_split "rn") and lo = x - hi exactly in fp32; the tensor core
// reads lo's top 11 significant bits.  Three integer / fp32 instructions per
// value (cvt.rna.tf32.f32 is four on its own, with an Inf / NaN guard the
// finite fields do not need).
struct AF {
    uint32_t h[4], l[4];
};

__device__ __forceinline__ void split1(AF &a, int i, float x) {
    const uint32_t hb = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
    a.h[i] = hb;
    a.l[i] = __float_as_uint(x - __uint_as_float(hb));
}

__device__ __forceinline__ void split2(AF &a, int i, float2 v) {
    split1(a, i, v.x);
    split1(a, i + 1, v.y);
}

// A fragment of element tile mt, k step ks (rows at x + k * KBS, elements g, g + 8
// at positions 16 mt + 2g, +1): a0 (g, t), a1 (g+8, t), a2 (g, t+4), a3 (g+8, t+4)
template <int KBS>
__device__ __forceinline__ void afrag(AF &a, const float *x, int mt, int ks, int lane) {
    const int g = lane >> 2, t = lane & 3;
    split2(a, 0, *reinterpret_cast<const float2 *>(x + (8 * ks + t) * KBS + 16 * mt + 2 * g));
    split2(a, 2, *reinterpret_cast<const float2 *>(x + (8 * ks + t + 4) * KBS + 16 * mt + 2 * g));
}

// the same fragment from pre-split hi / lo arrays
template <int KBS>
__device__ __forceinline__ void afrag_hl(AF &a, const float *xh, const float *xl, int mt, int ks, int lane) {
    const int g = lane >> 2, t = lane & 3;
    const int o0 = (8 * ks + t) * KBS + 16 * mt + 2 * g, o1 = o0 + 4 * KBS;
    const uint2 h0 = *reinterpret_cast<const uint2 *>(xh + o0), h1 = *reinterpret_cast<const uint2 *>(xh + o1);
    const uint2 l0 = *reinterpret_cast<const uint2 *>(xl + o0), l1 = *reinterpret_cast<const uint2 *>(xl + o1);
    a.h[0] = h0.x, a.h[1] = h0.y, a.h[2] = h1.x, a.h[3] = h1.y;
    a.l[0] = l0.x, a.l[1] = l0.y, a.l[2] = l1.x, a.l[3] = l1.y;
}

__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// d = A B from C = 0
__device__ __forceinline__ void hmma_z(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%10,%10,%10};\n"
        : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.0f));
}

// fresh = A B in split-TF32, small terms first
__device__ __forceinline__ void prod3(float (&d)[4], const AF &a, uint4 b) {
    hmma_z(d, a.l, b.x, b.y);
    hmma(d, a.h, b.z, b.w);
    hmma(d, a.h, b.x, b.y);
}

// the three split terms one at a time, so that a site issuing several
// independent products interleaves them (consecutive HMMAs independent)
__device__ __forceinline__ void term1(float (&d)[4], const AF &a, uint4 b) { hmma_z(d, a.l, b.x, b.y); }
__device__ __forceinline__ void term2(float (&d)[4], const AF &a, uint4 b) { hmma(d, a.h, b.z, b.w); }
__device__ __forceinline__ void term3(float (&d)[4], const AF &a, uint4 b) { hmma(d, a.h, b.x, b.y); }

// running sum += A B in split-TF32
__device__ __forceinline__ void prod3_acc(float (&d)[4], const AF &a, uint4 b) {
    hmma(d, a.l, b.x, b.y);
    hmma(d, a.h, b.z, b.w);
    hmma(d, a.h, b.x, b.y);
}

__device__ __forceinline__ void add4(float (&acc)[4], const float (&d)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += d[i];
}

__device__ __forceinline__ uint4 bfrag(const float *img, int idx, int lane) {
    return *reinterpret_cast<const uint4 *>(img + (size_t)(idx * 32 + lane) * 4);
}

template <int V>
struct IC {
    static constexpr int value = V;
};

// shared-memory position of element el (0..KB-1) of the CTA
__device__ __forceinline__ int epos(int el) { return (el & ~15) + 2 * (el & 7) + ((el >> 3) & 1); }

template <int N, bool SW>
__global__ void __launch_bounds__(CfgT<N, SW>::NTH, CfgT<N, SW>::MINB)
k_stage_tmma(const fused::FProb<float> P, const float *__restrict__ Qin, float *__restrict__ Qout,
             float *__restrict__ res, float tau_p, float tau_u, float a_rk, float b_rk, float dt, int block0) {
    using C = CfgT<N, SW>;
    constexpr int NP = C::NP, NPP = C::NPP, NQ = C::NQ, NQU = C::NQU, NFP = C::NFP, NFPK = C::NFPK, NFQ = C::NFQ;
    constexpr int NFQP = C::NFQP, NF = 4, FLD = 4, KB = C::KB, KBS = C::KBS, MT = C::MT, WPM = C::WPM;
    constexpr int QC = C::QC, QT = C::QT, JT = C::JT, FT = C::FT, RT = C::RT;

    static_assert(C::NTH == 256 && QC == 16 && KB == 32, "the volume epilogue maps 256 threads to 16 x 32 pairs");
    static_assert(C::WPM == 4 && C::NPROD % 4 == 0, "the point GEMMs are split between four warps per element tile");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw);
    float *sQ = reinterpret_cast<float *>(smem_raw + 16);
    float *ph = sQ + (size_t)FLD * NPP * KBS;
    // volume
    float *sVA = ph, *sVB = sVA + C::IMG_VA, *sW = sVB + C::IMG_VB;            // sW: [NWR][QC][KBS]
    // surface
    float *sP = ph;                                                            // [1 or 2][FLD][NFPK][KBS]
    float *sG = sP + (C::DBLP ? 2 : 1) * FLD * NFPK * KBS;                     // [FLD][NFQP][KBS]
    float *sVfi = sG + FLD * NFQP * KBS;
    float *sLift = sVfi + C::IMG_VFI;
    int32_t *sNbr = reinterpret_cast<int32_t *>(sLift + C::IMG_LIFT);
    int32_t *sCode = sNbr + NF * KB;
    int32_t *sFmask = sCode + NF * KB;
    int32_t *sExt = sFmask + NF * NFP;
    int32_t *sPerm = sExt + NF * 6 * NFP;
    // update
    // R split once into hi (over sQ, free after the surface) and lo parts
    float *sRh = sQ, *sRl = ph;                                                // [FLD][NPP][KBS]
    float *sU1 = sRl + FLD * NPP * KBS, *sU2 = sU1 + C::IMG_U1, *sW2 = sU2 + C::IMG_U2;   // sW2: [FLD][QC][KBS]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int mt = warp % MT, w0 = warp / MT;          // element tile; first n tile of this warp
    const int g = lane >> 2, tl = lane & 3;            // C fragment: rows g, g + 8; columns 2 tl, 2 tl + 1
    const int e0 = 16 * mt + g, e1 = e0 + 8;           // this lane's elements (C fragments)
    const int pe = 16 * mt + 2 * g;                    // their (adjacent) shared-memory positions
    const size_t S = P.Kpad;
    const size_t kblk = (size_t)(block0 + blockIdx.x) * KB;
    const float *ops = P.opVA;

    WADG_PROF_MARK(0);
    if (tid == 0) {
        fused::mbar_init(&bar[0], 1);    // "A" operator images (VA, Vfi / Pf, Vu)
        fused::mbar_init(&bar[1], 1);    // "B" operator images (VB, Pu)
    }
    uint32_t pa = 0, pb = 0;
    auto tma = [&](int k, float *dst, const float *src, int n) {   // thread 0 issues
        if (tid == 0) {
            fused::fence_proxy_async();
            fused::mbar_expect_tx(&bar[k], (uint32_t)(n * 4));
            fused::bulk_g2s(dst, src, (uint32_t)(n * 4), &bar[k]);
        }
    };
    auto twait = [&](int k) {
        uint32_t &phs = k ? pb : pa;
        fused::mbar_wait(&bar[k], phs);
        phs ^= 1u;
    };
    // chunk 0's volume operators land while the fields are staged
    tma(0, sVA, ops + C::O_VA, C::IMG_VA);
    tma(1, sVB, ops + C::O_VB, C::IMG_VB);
    // ---- fields -> sQ[c][j][pos(e)] (rows NP..NPP-1 zero): 16-byte loads of 4
    // elements, stored to their interleaved positions
    for (int r = tid; r < FLD * NPP * (KB / 4); r += C::NTH) {
        const int e4 = (r % (KB / 4)) * 4, row = r / (KB / 4);
        const int c = row / NPP, j = row % NPP;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < NP) v = __ldg(reinterpret_cast<const float4 *>(Qin + (size_t)(c * NP + j) * S + kblk + e4));
        float *dst = sQ + row * KBS;
        dst[epos(e4)] = v.x;
        dst[epos(e4 + 1)] = v.y;
        dst[epos(e4 + 2)] = v.z;
        dst[epos(e4 + 3)] = v.w;
    }
    // R accumulators (C fragments): field c, node tile jt = w0 + WPM * t
    float acc[RT][FLD][4];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
        for (int c = 0; c < FLD; ++c)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[t][c][i] = 0.f;
    __syncthreads();
    WADG_PROF_MARK(1);

    // C-fragment entry i: element e_i = i < 2 ? e0 : e1, column 2 tl + (i & 1)
    auto ent_e = [&](int i) { return i < 2 ? e0 : e1; };
    // 64-bit store of the two rows of column h (entries h, 2 + h) at row r of x
    auto st2 = [&](float *x, int r, float v0, float v1) {
        *reinterpret_cast<float2 *>(x + r * KBS + pe) = make_float2(v0, v1);
    };

    // ======================= volume =======================================
    // (chunk 0's operator images were issued before the fields)
    for (int ch = 0; ch < C::NCH; ++ch) {
        twait(0);
        // geometric factors of this thread's two (point, element) pairs of the
        // chunk epilogue below, loaded before the MMAs so that their latency overlaps
        float G[2][9];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = ch * QC + (tid >> 5) + 8 * h;
#pragma unroll
            for (int r = 0; r < 9; ++r) G[h][r] = q < NQ ? __ldg(P.geo + (size_t)(r * NQ + q) * S + kblk + lane) : 0.f;
        }
        // A (strong-weak): the chunk's point GEMMs, as products (operator, point tile):
        // D_r p, D_s p, D_t p, Vq u1, Vq u2, Vq u3 (-> sW rows 0..5) on both point
        // tiles.  The four warps of an element tile take consecutive runs of three, so
        // that each splits at most two field fragments per k step (p | p | u1, u2 |
        // u2, u3; one field per product group before: +1.7 % at N = 5); the products
        // of a k step are issued term by term.
        {
            auto phase_a = [&](auto wtag) {
                constexpr int W = decltype(wtag)::value;
                constexpr int PPW = C::NPROD / WPM;
                constexpr int F0 = C::prod_field(PPW * W), F1 = C::prod_field(PPW * W + PPW - 1);
                constexpr int N0 = C::prod_run(PPW * W, PPW);        // leading products on field F0
                float d[PPW][4];
#pragma unroll
                for (int k = 0; k < PPW; ++k)
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[k][i] = 0.f;
#pragma unroll 1
                for (int ks = 0; ks < NPP / 8; ++ks) {
                    AF x0, x1;
                    afrag<KBS>(x0, sQ + F0 * NPP * KBS, mt, ks, lane);
                    if constexpr (N0 < PPW) afrag<KBS>(x1, sQ + F1 * NPP * KBS, mt, ks, lane);
                    uint4 b[PPW];
                    float f[PPW][4];
#pragma unroll
                    for (int k = 0; k < PPW; ++k)
                        b[k] = bfrag(sVA, (C::prod_op(PPW * W + k) * (NPP / 8) + ks) * QT + C::prod_qt(PPW * W + k), lane);
#pragma unroll
                    for (int k = 0; k < N0; ++k) term1(f[k], x0, b[k]);
#pragma unroll
                    for (int k = N0; k < PPW; ++k) term1(f[k], x1, b[k]);
#pragma unroll
                    for (int k = 0; k < N0; ++k) term2(f[k], x0, b[k]);
#pragma unroll
                    for (int k = N0; k < PPW; ++k) term2(f[k], x1, b[k]);
#pragma unroll
                    for (int k = 0; k < N0; ++k) term3(f[k], x0, b[k]);
#pragma unroll
                    for (int k = N0; k < PPW; ++k) term3(f[k], x1, b[k]);
#pragma unroll
                    for (int k = 0; k < PPW; ++k) add4(d[k], f[k]);
                }
#pragma unroll
                for (int k = 0; k < PPW; ++k)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        st2(sW, C::prod_row(PPW * W + k) * QC + 8 * C::prod_qt(PPW * W + k) + 2 * tl + h, d[k][h],
                            d[k][2 + h]);
            };
            if constexpr (SW) {
                switch (w0) {
                    case 0: phase_a(IC<0>{}); break;
                    case 1: phase_a(IC<1>{}); break;
                    case 2: phase_a(IC<2>{}); break;
                    default: phase_a(IC<3>{}); break;
                }
            }
        }
        if constexpr (!SW) {
            // strong form: units (point tile, field c), du_a,c = D_a Q_c -> sW rows
            // 3 c + a (one field per unit measured faster than one field per warp here)
#pragma unroll
            for (int t = 0; t < C::AU; ++t) {
                const int u = w0 + WPM * t;
                if (u >= C::NAU) continue;
                const int qt = u % QT, c = u / QT;
                float d[3][4];
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[m][i] = 0.f;
#pragma unroll 1
                for (int ks = 0; ks < NPP / 8; ++ks) {
                    AF x;
                    afrag<KBS>(x, sQ + c * NPP * KBS, mt, ks, lane);
                    uint4 b[3];
                    float f[3][4];
#pragma unroll
                    for (int m = 0; m < 3; ++m) b[m] = bfrag(sVA, (m * (NPP / 8) + ks) * QT + qt, lane);
#pragma unroll
                    for (int m = 0; m < 3; ++m) term1(f[m], x, b[m]);
#pragma unroll
                    for (int m = 0; m < 3; ++m) term2(f[m], x, b[m]);
#pragma unroll
                    for (int m = 0; m < 3; ++m) term3(f[m], x, b[m]);
#pragma unroll
                    for (int m = 0; m < 3; ++m) add4(d[m], f[m]);
                }
#pragma unroll
                for (int m = 0; m < 3; ++m)
#pragma unroll
                    for (int h = 0; h < 2; ++h) st2(sW, (3 * c + m) * QC + 8 * qt + 2 * tl + h, d[m][h], d[m][2 + h]);
            }
        }
        __syncthreads();
        // epilogue, one thread per (point, element) pair, in place: gp_i = sum_a G_ai dp_a
        // and F_a = sum_i G_ai U_i (the quadrature weight is folded into DTW), or for the
        // strong form gp_i and div = sum_i sum_a G_ai du_a,i (R/pkg/src/wadg/solver.py:259-264)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float *w = sW + ((tid >> 5) + 8 * h) * KBS + epos(lane);
            const float *g = G[h];
            const float d0 = w[0], d1 = w[QC * KBS], d2 = w[2 * QC * KBS];
            if constexpr (SW) {
                const float u0 = w[3 * QC * KBS], u1 = w[4 * QC * KBS], u2 = w[5 * QC * KBS];
#pragma unroll
                for (int i = 0; i < 3; ++i) w[i * QC * KBS] = g[0 * 3 + i] * d0 + g[1 * 3 + i] * d1 + g[2 * 3 + i] * d2;
#pragma unroll
                for (int a = 0; a < 3; ++a)
                    w[(3 + a) * QC * KBS] = g[a * 3 + 0] * u0 + g[a * 3 + 1] * u1 + g[a * 3 + 2] * u2;
            } else {
                float du[3][3];                  // [field i][a]
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int a = 0; a < 3; ++a) du[i][a] = w[(3 * (1 + i) + a) * QC * KBS];
                float div = 0.f;
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    div += g[0 * 3 + i] * du[i][0] + g[1 * 3 + i] * du[i][1] + g[2 * 3 + i] * du[i][2];
#pragma unroll
                for (int i = 0; i < 3; ++i) w[i * QC * KBS] = g[0 * 3 + i] * d0 + g[1 * 3 + i] * d1 + g[2 * 3 + i] * d2;
                w[3 * QC * KBS] = div;
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCH) tma(0, sVA, ops + C::O_VA + (size_t)(ch + 1) * C::IMG_VA, C::IMG_VA);
        twait(1);
        // B: R_p += sum_a DTW_a F_a (strong: (-Pq) div), R_u_i += (-Pq) gp_i
        if constexpr (!SW) {
#pragma unroll
            for (int ks = 0; ks < QC / 8; ++ks) {
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    AF w;
                    afrag<KBS>(w, sW + (c == 0 ? 3 : c - 1) * QC * KBS, mt, ks, lane);
#pragma unroll
                    for (int t = 0; t < RT; ++t) {
                        const int jt = w0 + WPM * t;
                        if (jt < JT) {
                            float f[4];
                            prod3(f, w, bfrag(sVB, ks * JT + jt, lane));
                            add4(acc[t][c], f);
                        }
                    }
                }
            }
        } else
#pragma unroll
        for (int ks = 0; ks < QC / 8; ++ks) {
            float fp[RT][4];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                AF w;
                afrag<KBS>(w, sW + (3 + a) * QC * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int jt = w0 + WPM * t;
                    if (jt < JT) {
                        const uint4 b = bfrag(sVB, (a * (QC / 8) + ks) * JT + jt, lane);
                        if (a == 0)
                            prod3(fp[t], w, b);
                        else
                            prod3_acc(fp[t], w, b);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < RT; ++t)
                if (w0 + WPM * t < JT) add4(acc[t][0], fp[t]);
#pragma unroll
            for (int i3 = 0; i3 < 3; ++i3) {
                AF w;
                afrag<KBS>(w, sW + i3 * QC * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int jt = w0 + WPM * t;
                    if (jt < JT) {
                        float f[4];
                        prod3(f, w, bfrag(sVB, (3 * (QC / 8) + ks) * JT + jt, lane));
                        add4(acc[t][1 + i3], f);
                    }
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
    tma(0, sVfi, ops + C::O_VFI, C::IMG_VFI);   // stays for the whole surface
    twait(0);
    __syncthreads();
    // exterior face-node values of face f -> buf[c][i][pos(e)] (rows NFP..NFPK-1 zero)
    auto gather = [&](int f, float *buf) {
        for (int r = tid; r < FLD * NFPK * KB; r += C::NTH) {
            const int el = r % KB, rest = r / KB;
            const int i = rest % NFPK, c = rest / NFPK;
            float *dst = buf + (c * NFPK + i) * KBS + epos(el);
            if (i >= NFP) {
                *dst = 0.f;
                continue;
            }
            const int nb = sNbr[f * KB + el];
            const int code = sCode[f * KB + el];
            if (nb >= 0) {
                fused::cp_async_elem(dst, Qin + (size_t)(c * NP + sExt[code * NFP + i]) * S + nb);
            } else if (nb == -1) {       // mirror BC (solver.py:214-217): p+ = -p-, u+ = u-
                const float m = sQ[(c * NPP + sFmask[f * NFP + i]) * KBS + epos(el)];
                *dst = (c == 0) ? -m : m;
            } else {
                fused::cp_async_elem(dst, P.halo + ((size_t)(-nb - 2) * FLD + c) * NFP + sPerm[(code % P.nor) * NFP + i]);
            }
        }
        fused::cp_async_commit();
    };
    gather(0, sP);
    for (int f = 0; f < NF; ++f) {
        float *cur = C::DBLP ? sP + (f & 1) * (FLD * NFPK * KBS) : sP;
        if (C::DBLP && f + 1 < NF) {
            gather(f + 1, sP + ((f + 1) & 1) * (FLD * NFPK * KBS));
            fused::cp_async_wait<1>();
        } else {
            fused::cp_async_wait<0>();
        }
        tma(0, sLift, ops + C::O_LIFT + (size_t)f * C::IMG_LIFT, C::IMG_LIFT);   // lands during the traces
        __syncthreads();
        // traces at the face points (own from sQ's face nodes, exterior from cur), then the flux
#pragma unroll 1
        for (int t = 0; t < C::TT; ++t) {
            const int ft = w0 + WPM * t;
            if (ft >= FT) continue;
            float fgv[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int fq = 8 * ft + 2 * tl + (i & 1);
                const size_t o = (size_t)(f * NFQ + fq) * S + kblk + ent_e(i);
#pragma unroll
                for (int dd = 0; dd < 4; ++dd) fgv[i][dd] = fq < NFQ ? __ldg(P.fgeo + (size_t)dd * NFQT * S + o) : 0.f;
            }
            float dm[FLD][4], dp[FLD][4];
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int i = 0; i < 4; ++i) dm[c][i] = dp[c][i] = 0.f;
#pragma unroll
            for (int ks = 0; ks < NFPK / 8; ++ks) {
                const int i0 = 8 * ks + tl, i1 = i0 + 4;
                const int n0 = i0 < NFP ? sFmask[f * NFP + i0] : -1;
                const int n1 = i1 < NFP ? sFmask[f * NFP + i1] : -1;
                const uint4 b = bfrag(sVfi, ks * FT + ft, lane);
#pragma unroll
                for (int c = 0; c < FLD; ++c) {
                    AF xm, xp;
                    const float2 z2 = make_float2(0.f, 0.f);
                    const float2 m0 = n0 >= 0 ? *reinterpret_cast<const float2 *>(sQ + (c * NPP + n0) * KBS + pe) : z2;
                    const float2 m1 = n1 >= 0 ? *reinterpret_cast<const float2 *>(sQ + (c * NPP + n1) * KBS + pe) : z2;
                    split2(xm, 0, m0);
                    split2(xm, 2, m1);
                    split2(xp, 0, *reinterpret_cast<const float2 *>(cur + (c * NFPK + i0) * KBS + pe));
                    split2(xp, 2, *reinterpret_cast<const float2 *>(cur + (c * NFPK + i1) * KBS + pe));
                    float f4[4];
                    prod3(f4, xm, b);
                    add4(dm[c], f4);
                    prod3(f4, xp, b);
                    add4(dp[c], f4);
                }
            }
            float gv[FLD][4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float n0 = fgv[i][0], n1 = fgv[i][1], n2 = fgv[i][2], sJh = fgv[i][3];
                const float djp = dp[0][i] - dm[0][i];
                const float dUn = (dp[1][i] - dm[1][i]) * n0 + (dp[2][i] - dm[2][i]) * n1 + (dp[3][i] - dm[3][i]) * n2;
                const float avg = (dp[1][i] + dm[1][i]) * n0 + (dp[2][i] + dm[2][i]) * n1 + (dp[3][i] + dm[3][i]) * n2;
                const float fpp = (SW ? avg : dUn) - tau_p * djp;   // strong: [u.n] (solver.py:220-232)
                const float fuu = djp - tau_u * dUn;
                // padded face points have zero factors, hence zero flux
                gv[0][i] = fpp * sJh;
                gv[1][i] = fuu * (sJh * n0);
                gv[2][i] = fuu * (sJh * n1);
                gv[3][i] = fuu * (sJh * n2);
            }
#pragma unroll
            for (int c = 0; c < FLD; ++c)
#pragma unroll
                for (int h = 0; h < 2; ++h) st2(sG, c * NFQP + 8 * ft + 2 * tl + h, gv[c][h], gv[c][2 + h]);
        }
        __syncthreads();
        if (!C::DBLP && f + 1 < NF) gather(f + 1, sP);   // the traces are done with the buffer
        // L2 prefetches of the next face's factors (loaded before its trace MMAs) and,
        // below, of the rows the LSRK write reads: N = 6 / 7 +1.5 / +0.8 %, but
        // N = 5 -5.5 % (two CTAs per SM there already hide the latency)
        if (N >= 6 && f + 1 < NF)
            for (int r = tid; r < 4 * NFQ; r += C::NTH)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(P.fgeo + (size_t)(r / NFQ) * NFQT * S +
                                                            (size_t)((f + 1) * NFQ + r % NFQ) * S + kblk));
        twait(0);
        // lift: R_c += (-Pf_f) g_c
#pragma unroll 1
        for (int ks = 0; ks < NFQP / 8; ++ks) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                AF gvf;
                afrag<KBS>(gvf, sG + c * NFQP * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int jt = w0 + WPM * t;
                    if (jt < JT) {
                        float f4[4];
                        prod3(f4, gvf, bfrag(sLift, ks * JT + jt, lane));
                        add4(acc[t][c], f4);
                    }
                }
            }
        }
        __syncthreads();
    }

    // ======================= WADG update + LSRK ===========================
    WADG_PROF_MARK(3);
    tma(0, sU1, ops + C::O_U1, C::IMG_U1);
    tma(1, sU2, ops + C::O_U2, C::IMG_U2);
    // L2 prefetch of this tile's Q_in and old res rows, read by the LSRK write
    if (N >= 6)
    for (int r = tid; r < 2 * FLD * NP; r += C::NTH) {
        const float *base = r < FLD * NP ? Qin : res;
        if (r < FLD * NP || a_rk != 0.f)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(base + (size_t)(r % (FLD * NP)) * S + kblk));
    }
    // R -> sRh / sRl[c][j][pos(e)] (the A operand of z = Vu R, split once);
    // accumulators restart at zero.  sQ is overwritten: the LSRK write re-reads Q_in.
    __syncthreads();
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int jt = w0 + WPM * t;
        if (jt < JT) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    AF sp;
                    split2(sp, 0, make_float2(acc[t][c][h], acc[t][c][2 + h]));
                    st2(sRh, c * NPP + 8 * jt + 2 * tl + h, __uint_as_float(sp.h[0]), __uint_as_float(sp.h[1]));
                    st2(sRl, c * NPP + 8 * jt + 2 * tl + h, __uint_as_float(sp.l[0]), __uint_as_float(sp.l[1]));
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[t][c][i] = 0.f;
            }
        }
    }
    __syncthreads();
    for (int ch = 0; ch < C::NCHU; ++ch) {
        twait(0);
        // z_c = Vu R_c at point tile qt for the field pair pr, times c^2/J (p) or 1/J (u)
#pragma unroll
        for (int t = 0; t < C::ZU; ++t) {
            const int u = w0 + WPM * t;
            if (u >= 2 * QT) continue;
            const int qt = u % QT, pr = u / QT;
            float wu[4], wp[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int q = ch * QC + 8 * qt + 2 * tl + (i & 1);
                const bool ok = q < NQU;
                wu[i] = ok ? __ldg(P.wu + (size_t)q * S + kblk + ent_e(i)) : 0.f;
                wp[i] = (ok && P.wp && pr == 0) ? __ldg(P.wp + (size_t)q * S + kblk + ent_e(i)) : 0.f;
            }
            float z[2][4];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                for (int i = 0; i < 4; ++i) z[cc][i] = 0.f;
#pragma unroll 1
            for (int ks = 0; ks < NPP / 8; ++ks) {
                const uint4 b = bfrag(sU1, ks * QT + qt, lane);
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    AF x;
                    afrag_hl<KBS>(x, sRh + (2 * pr + cc) * NPP * KBS, sRl + (2 * pr + cc) * NPP * KBS, mt, ks, lane);
                    float f4[4];
                    prod3(f4, x, b);
                    add4(z[cc], f4);
                }
            }
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int c = 2 * pr + cc;
                float v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = (c == 0 ? (P.wp ? wp[i] : P.c2 * wu[i]) : wu[i]) * z[cc][i];
#pragma unroll
                for (int h = 0; h < 2; ++h) st2(sW2, c * QC + 8 * qt + 2 * tl + h, v[h], v[2 + h]);
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCHU) tma(0, sU1, ops + C::O_U1 + (size_t)(ch + 1) * C::IMG_U1, C::IMG_U1);
        twait(1);
        // R'_c += Pu (omega z_c)
#pragma unroll
        for (int ks = 0; ks < QC / 8; ++ks) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                AF wv;
                afrag<KBS>(wv, sW2 + c * QC * KBS, mt, ks, lane);
#pragma unroll
                for (int t = 0; t < RT; ++t) {
                    const int jt = w0 + WPM * t;
                    if (jt < JT) {
                        float f4[4];
                        prod3(f4, wv, bfrag(sU2, ks * JT + jt, lane));
                        add4(acc[t][c], f4);
                    }
                }
            }
        }
        __syncthreads();
        if (ch + 1 < C::NCHU) tma(1, sU2, ops + C::O_U2 + (size_t)(ch + 1) * C::IMG_U2, C::IMG_U2);
    }
    WADG_PROF_MARK(4);
    // res = a res + dt Minv(rhs); Q_out = Q_in + b res (entries: elements e0 / e1, nodes 8 jt + 2 tl + h)
#pragma unroll
    for (int t = 0; t < RT; ++t) {
        const int jt = w0 + WPM * t;
        if (jt < JT) {
#pragma unroll
            for (int c = 0; c < FLD; ++c) {
                float rold[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 8 * jt + 2 * tl + (i & 1);
                    rold[i] = (a_rk != 0.f && j < NP) ? __ldg(res + (size_t)(c * NP + j) * S + kblk + ent_e(i)) : 0.f;
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int j = 8 * jt + 2 * tl + (i & 1);
                    if (j < NP) {
                        const size_t o = (size_t)(c * NP + j) * S + kblk + ent_e(i);
                        const float r = a_rk * rold[i] + dt * acc[t][c][i];
                        res[o] = r;
                        Qout[o] = __ldg(Qin + o) + b_rk * r;
                    }
                }
            }
        }
    }
    __syncthreads();
    WADG_PROF_MARK(5);
}

}  // namespace tk
}  // namespace wadg
